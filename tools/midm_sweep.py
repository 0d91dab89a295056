"""Mid-M schedule sweep of the tcgen05 tree GEMM (pure scheduling knobs, same bits):
Llama down_proj K=14336 N=4096 and o_proj K=4096 N=4096 at M = 256..2048; device time
per call from a CUDA graph of 10 calls rotating 3 weight copies.
usage: python tools/midm_sweep.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

from tools.timing import graph_time  # noqa: E402

cfg = tb.BlockConfig(64, 256, 128, 0)
# schedule knobs (tbik_set_schedule): pure scheduling, the same bits ('!' marks a violation)
VARIANTS = [("default", {}), ("units2", {"tc_units": 2}), ("units4", {"tc_units": 4}), ("deep0", {"tc_deep": 0}),
            ("deep1", {"tc_deep": 1}), ("gm4", {"tc_group_m": 4})]


for K, N in ((14336, 4096), (4096, 4096), (4096, 28672)):
    ws = [torch.randn(K, N, device="cuda").to(torch.bfloat16) for _ in range(3)]
    for M in (256, 512, 768, 1024, 1536, 2048, 4096):
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda")
        ref = None
        line = [f"K={K} N={N} M={M:5d}"]
        for name, knobs in VARIANTS:
            f = lambda i: tb.tree_matmul(x, ws[i], cfg, tb.LEAF_TCGEN05, out=y)  # noqa: E731
            with tb.schedule(**knobs):
                t = graph_time(f)
            if ref is None:
                ref = y.clone()
            same = torch.equal(ref.view(torch.int32), y.view(torch.int32))
            line.append(f"{name} {2 * M * K * N / t / 1e6:6.0f}{'' if same else '!'}")
        yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t = graph_time(lambda i: torch.matmul(x, ws[i], out=yb))
        line.append(f"cublas {2 * M * K * N / t / 1e6:6.0f} TFLOP/s")
        print(" | ".join(line), flush=True)
