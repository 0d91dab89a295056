"""Exact-leaf (TBIK_LEAF_FMA) GEMM throughput, v2 vs v1 kernel (TBIK_FMA_V1), same bits."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from tools.tune_tc import timeit  # noqa: E402

K, N = 14336, 4096
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
cfg = tb.BlockConfig(64, 256, 128, 0)
for M in (64, 256, 1024, 4096):
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    outs = []
    for v1 in ("", "1"):
        if v1:
            os.environ["TBIK_FMA_V1"] = "1"
        else:
            os.environ.pop("TBIK_FMA_V1", None)
        ms = timeit(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_FMA), 3)
        outs.append(tb.tree_matmul(x, w, cfg, tb.LEAF_FMA))
        print(f"M={M} {'v1' if v1 else 'v2'}: {ms*1e3:9.1f} us {2*M*N*K/ms/1e9:6.1f} TFLOP/s", flush=True)
    print("   bits equal:", torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32)), flush=True)
