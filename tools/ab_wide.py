"""A/B the 256x128 and 256x256 tcgen05 TBIK kernels (same bits) at several M."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from tools.tune_tc import timeit  # noqa: E402

for K, N in ((14336, 4096), (4096, 28672), (4096, 6144)):
    w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    for M in (int(a) for a in (sys.argv[1:] or ["256", "1024", "4096"])):
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda")
        outs = {}
        for wide in ("0", "1"):
            os.environ["TBIK_TC_WIDE"] = wide
            ms = timeit(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y), 10)
            outs[wide] = y.clone()
            print(f"K={K} N={N} M={M} wide={wide}: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s", flush=True)
        print("   bits equal:", torch.equal(outs["0"].view(torch.int32), outs["1"].view(torch.int32)), flush=True)
        yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ms = timeit(lambda: torch.matmul(x, w, out=yb), 10)
        print(f"K={K} N={N} M={M} cuBLAS: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s", flush=True)
