"""256 x 192 pair tiles (tbik_gemm_tc_w192.cu) vs the 256 x 128 kernel: bit equality on
ragged / split / k_first = 1 / TP-shard shapes, then device time per call (CUDA
events, 20 back-to-back calls) for the schedule variants.
usage: python tools/wide_check.py [check] [time] [M K N ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402


def ev_time(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def run(x, w, cfg, knobs):
    with tb.schedule(**knobs):
        y = tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05)
    torch.cuda.synchronize()
    return y


def check():
    g = torch.Generator(device="cuda").manual_seed(7)
    cases = [  # M, K, N, block_k, k_first, knobs
        (512, 14336, 512, 256, 0, {}),
        (1024, 4096, 1024, 256, 0, {}),          # k_first = 1 (16 groups)
        (300, 2048, 200, 256, 0, {}),            # ragged M and N
        (777, 3000, 520, 256, 0, {}),            # ragged K (partial last leaf)
        (1024, 14336, 4096, 256, 0, {"tc_units": 2}),
        (1024, 14336, 4096, 256, 0, {"tc_units": 4}),
        (4096, 14336, 4096, 256, 0, {}),
        (4096, 14336, 4096, 256, 0, {"tc_wide_tail": 0}),
        (4096, 4096, 4096, 256, 0, {}),
        (2048, 1792, 4096, 256, 0, {}),          # TP = 8 shard view (one group)
        (1536, 8192, 1280, 128, 0, {}),          # block_k = 128
        (1024, 6144, 768, 320, 0, {}),           # block_k = 320
        (640, 4096, 2304, 256, 4, {}),           # explicit k_first
        (2048, 25600, 5120, 128, 0, {}),         # Qwen3-32B down_proj
        (1000, 4096, 4000, 256, 0, {}),          # N not a multiple of 192 / 96
        (2048, 14336, 4096, 256, 0, {"tc_units": 2}),
    ]
    ok = True
    for M, K, N, bk, kf, knobs in cases:
        x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
        w = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
        cfg = tb.BlockConfig(64, bk, 128, kf)
        ref = run(x, w, cfg, {"tc_wide": 0, **{k: v for k, v in knobs.items() if k == "tc_units"}})
        res = []
        for name, kv in (("w192", {"tc_wide": 1}),):
            y = run(x, w, cfg, {**kv, **knobs})
            same = torch.equal(ref.view(torch.int32), y.view(torch.int32))
            ok &= same
            nbad = int((ref.view(torch.int32) != y.view(torch.int32)).sum())
            res.append(f"{name} {'bit-identical' if same else f'DIFFER ({nbad})'}")
        print(f"M={M} K={K} N={N} bk={bk} kf={kf} {knobs}: {' | '.join(res)}", flush=True)
    print("ALL BIT-IDENTICAL" if ok else "MISMATCH", flush=True)
    return ok


SHAPES = [(4096, 14336, 4096), (2048, 14336, 4096), (1024, 14336, 4096), (512, 14336, 4096),
          (4096, 7168, 4096), (4096, 3584, 4096), (4096, 1792, 4096), (1024, 1792, 4096),
          (4096, 4096, 4096), (2048, 4096, 4096), (4096, 4096, 28672), (1024, 4096, 6144),
          (1024, 25600, 5120), (2048, 25600, 5120), (4096, 25600, 5120), (4096, 5120, 10240), (2048, 3200, 5120)]
MID_VARIANTS = [("narrow", {"tc_wide": 0}), ("w192", {"tc_wide": 1}), ("w192_u1", {"tc_wide": 1, "tc_units": 1}),
                ("w192_u2", {"tc_wide": 1, "tc_units": 2}), ("w192_u4", {"tc_wide": 1, "tc_units": 4})]
VARIANTS = MID_VARIANTS if os.environ.get("MID") else [
    ("narrow", {"tc_wide": 0}), ("w192", {"tc_wide": 1}), ("w192_notail", {"tc_wide": 1, "tc_wide_tail": 0}),
    ("w192_gm4", {"tc_wide": 1, "tc_group_m": 4})]


def timing(shapes):
    for M, K, N in shapes:
        bk = 256 if K % 256 == 0 and K != 25600 else 128
        cfg = tb.BlockConfig(64, bk, 128, 0)
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda")
        ref = None
        line = [f"M={M} K={K} N={N}"]
        for name, knobs in VARIANTS:
            with tb.schedule(**knobs):
                t = ev_time(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y))
            same = True if ref is None else torch.equal(ref.view(torch.int32), y.view(torch.int32))
            if ref is None:
                ref = y.clone()
            line.append(f"{name} {t:7.1f} us {2 * M * K * N / t / 1e6:6.0f} TF{'' if same else ' BITS DIFFER'}")
        yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t = ev_time(lambda: torch.matmul(x, w, out=yb))
        line.append(f"cublas {t:7.1f} us {2 * M * K * N / t / 1e6:6.0f} TF")
        print(" | ".join(line), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    do_check = "check" in args or not any(a in ("check", "time") for a in args)
    do_time = "time" in args or not any(a in ("check", "time") for a in args)
    nums = [int(a) for a in args if a.isdigit()]
    shapes = [tuple(nums[i:i + 3]) for i in range(0, len(nums), 3)] if nums else SHAPES
    if do_check and not check():
        sys.exit(1)
    if do_time:
        timing(shapes)
