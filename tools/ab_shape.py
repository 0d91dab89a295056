"""Time one TBIK GEMM shape under the current environment knobs (run once per
knob setting: the launcher reads TBIK_TC_* once per process).
usage: ab_shape.py label M K N [M K N ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from tools.tune_tc import timeit  # noqa: E402

label = sys.argv[1]
dims = [int(a) for a in sys.argv[2:]]
cfg = tb.BlockConfig(64, 256, 128, 0)
for i in range(0, len(dims), 3):
    M, K, N = dims[i:i + 3]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    ms = timeit(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y), 20)
    h = int(y.view(torch.int32).to(torch.int64).sum().item())
    print(f"{label} M={M} K={K} N={N}: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s bits={h:#x}", flush=True)
