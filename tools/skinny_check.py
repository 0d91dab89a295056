"""Swap-AB skinny tcgen05 kernel (tbik_gemm_skinny.cu) vs the wide tcgen05 kernel:
bit identity over decode-sized shapes, then timing with W evicted from L2.
usage: python tools/skinny_check.py [--time-only]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

torch.manual_seed(0)
cfg = tb.BlockConfig(64, 256, 128, 0)


def run(x, w, skinny, **env):
    os.environ["TBIK_TC_SKINNY"] = "1" if skinny else "0"
    for k, v in env.items():
        os.environ[k] = str(v)
    y = tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05)
    for k in env:
        del os.environ[k]
    return y


def same(a, b):
    return torch.equal(a.view(torch.int32), b.view(torch.int32))


if "--time-only" not in sys.argv:
    shapes = [(1, 14336, 4096), (2, 14336, 4096), (5, 14336, 4096), (16, 14336, 4096), (17, 14336, 4096),
              (32, 14336, 4096), (33, 14336, 4096), (64, 14336, 4096), (65, 14336, 4096), (128, 14336, 4096), (100, 4096, 1000), (16, 1792, 4096), (16, 3584, 4096),
              (8, 4096, 4096), (16, 1000, 1000), (3, 777, 300), (64, 25600 // 8 * 8, 5120), (16, 8192, 1024)]
    ok_all = True
    for (M, K, N) in shapes:
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
        ref = run(x, w, False)
        outs = {"default": run(x, w, True)}
        plan = tb.plan_blocks(K, cfg, 1)
        L = plan.leaves
        u = 1
        while u <= L:
            outs[f"units={u}"] = run(x, w, True, TBIK_SK_UNITS=u, TBIK_SK_LEAF=0)
            u *= 2
        if plan.k_first > 1 and plan.tiles_total <= 8:
            outs["leaf"] = run(x, w, True, TBIK_SK_LEAF=1)
        res = {k: same(v, ref) for k, v in outs.items()}
        ok = all(res.values())
        ok_all &= ok
        f64 = (x.double() @ w.double())
        err = ((outs["default"].double() - f64).abs().max() / f64.abs().max()).item()
        print(f"M={M} K={K} N={N} T={plan.tiles_total} kf={plan.k_first} L={L}: "
              f"{'OK' if ok else 'MISMATCH'} {res} relerr_vs_f64={err:.2e}", flush=True)
    # TP shards through the row-parallel API (views of K, global k_first)
    x = torch.randn(16, 14336, device="cuda").to(torch.bfloat16)
    w = torch.randn(14336, 4096, device="cuda").to(torch.bfloat16)
    os.environ["TBIK_TC_SKINNY"] = "0"
    ref = tb.row_parallel_forward(x, w, tb.DeviceGroup(1), cfg, 8, tb.LEAF_TCGEN05)
    os.environ["TBIK_TC_SKINNY"] = "1"
    for tp in (1, 2, 4, 8):
        y = tb.row_parallel_forward(x, w, tb.DeviceGroup(tp), cfg, 8, tb.LEAF_TCGEN05)
        print(f"row-parallel M=16 tp={tp}: {'OK' if same(y, ref) else 'MISMATCH'}", flush=True)
        ok_all &= same(y, ref)
    print("ALL_BITS_EQUAL" if ok_all else "SOME_MISMATCH", flush=True)

# timing (W evicted from L2 before each call)
# eviction by READING 256 MB (a write-flush would leave dirty lines whose write-back
# competes with the weight stream)
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")
K, N = 14336, 4096
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)


def timeit(fn, reps=20):
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=sink)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for M in (1, 16, 64, 128):
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    line = [f"M={M}"]
    for name, env in [("wide", {"TBIK_TC_SKINNY": "0"}), ("skinny", {"TBIK_TC_SKINNY": "1"})] + \
            [(f"sk_u{u}", {"TBIK_TC_SKINNY": "1", "TBIK_SK_UNITS": str(u), "TBIK_SK_LEAF": "0"}) for u in (1, 2, 4, 8)]:
        os.environ.update(env)
        t = timeit(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y))
        for k in env:
            del os.environ[k]
        line.append(f"{name} {t:6.1f}us ({K * N * 2 / t / 1e3:5.0f} GB/s W)")
    t = timeit(lambda: torch.matmul(x, w, out=yb))
    line.append(f"cublas {t:6.1f}us")
    print(" | ".join(line), flush=True)
# TP=8 shard at decode size (K=1792, global k_first 7)
x = torch.randn(16, K, device="cuda").to(torch.bfloat16)
for name, env in [("wide", {"TBIK_TC_SKINNY": "0"}), ("skinny", {"TBIK_TC_SKINNY": "1"}),
                  ("sk_leaf0", {"TBIK_TC_SKINNY": "1", "TBIK_SK_LEAF": "0"})]:
    os.environ.update(env)
    g = tb.DeviceGroup(8)
    t = timeit(lambda: tb.row_parallel_forward(x, w, g, cfg, 8, tb.LEAF_TCGEN05))
    for k in env:
        del os.environ[k]
    print(f"simulated TP=8 row-parallel M=16 (8 shard GEMMs + tree AR) {name}: {t:6.1f}us", flush=True)
