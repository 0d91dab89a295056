"""A/B of schedule knobs on the tcgen05 tree GEMM (same bits, checked): device time
per call with CUDA events, 20 back-to-back calls (inputs resident; the bench shape's
operands exceed L2).  usage: python tools/ab_knobs.py [M K N ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

SHAPES = [(4096, 14336, 4096), (2048, 14336, 4096), (1024, 14336, 4096), (4096, 4096, 4096), (4096, 4096, 28672),
          (2048, 25600, 5120)]
VARIANTS = [("default", {}), ("deep1", {"tc_deep": 1}), ("deep0", {"tc_deep": 0})]


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


args = [int(a) for a in sys.argv[1:]]
shapes = [tuple(args[i:i + 3]) for i in range(0, len(args), 3)] if args else SHAPES
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
