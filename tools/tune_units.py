"""Time the tcgen05 TBIK GEMM for each K-split factor (TBIK_TC_UNITS) at several M."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from tools.tune_tc import timeit  # noqa: E402

K, N = 14336, 4096
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
cfg = tb.BlockConfig(64, 256, 128, 0)
for M in (int(a) for a in (sys.argv[1:] or ["64", "256", "1024", "4096"])):
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    ref = None
    for u in ("1", "2", "4", "8"):
        os.environ["TBIK_TC_UNITS"] = u
        ms = timeit(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y), 20)
        ref = y.clone() if ref is None else ref
        same = torch.equal(ref.view(torch.int32), y.view(torch.int32))
        print(f"M={M} units={u}: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s bits_equal={same}", flush=True)
    os.environ.pop("TBIK_TC_UNITS")
    yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda: torch.matmul(x, w, out=yb), 20)
    print(f"M={M} cuBLAS: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s", flush=True)
