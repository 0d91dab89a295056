"""Skinny-kernel unit / tile-width choice on Qwen3-32B decode shapes (M = 16): device
time per call from a CUDA graph of 20 calls rotating 3 weight copies.
usage: python tools/skinny_units.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

cfg = tb.BlockConfig(64, 256, 128, 0)


def graph_time(fn, reps=20):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i % 3)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / (5 * reps)


for (K, N) in ((8192, 5120), (25600, 5120), (5120, 10240), (4096, 6144), (14336, 4096)):
    ws = [torch.randn(K, N, device="cuda").to(torch.bfloat16) for _ in range(3)]
    x = torch.randn(16, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(16, N, device="cuda")
    line = [f"K={K} N={N}"]
    for name, env in (("default", {}), ("u1", {"TBIK_SK_UNITS": "1"}), ("u2", {"TBIK_SK_UNITS": "2"}),
                      ("u4", {"TBIK_SK_UNITS": "4"}), ("bn64", {"TBIK_SK_BN": "64"}),
                      ("bn64u2", {"TBIK_SK_BN": "64", "TBIK_SK_UNITS": "2"})):
        for k in ("TBIK_SK_UNITS", "TBIK_SK_BN"):
            os.environ.pop(k, None)
        os.environ.update(env)
        t = graph_time(lambda i: tb.tree_matmul(x, ws[i], cfg, tb.LEAF_TCGEN05, out=y))
        line.append(f"{name} {t:5.1f}")
    for k in ("TBIK_SK_UNITS", "TBIK_SK_BN"):
        os.environ.pop(k, None)
    yb = torch.empty(16, N, device="cuda", dtype=torch.bfloat16)
    line.append(f"cublas {graph_time(lambda i: torch.matmul(x, ws[i], out=yb)):5.1f} us  (W {K * N * 2 / 1e6:.0f} MB)")
    print(" | ".join(line), flush=True)
