"""Time the tcgen05 TBIK GEMM for the merge-warp variants selected by
TBIK_TC_EPI / TBIK_TC_LB (read once per process; run one process per variant).
Prints TFLOP/s and a bit checksum per shape so variants can be compared."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from tools.tune_tc import timeit  # noqa: E402

tag = f"epi={os.environ.get('TBIK_TC_EPI', '4')} lb={os.environ.get('TBIK_TC_LB', '1')}"
g = torch.Generator(device="cuda").manual_seed(1)
for K, N in ((14336, 4096), (4096, 28672), (4096, 6144), (4096, 128256)):
    w = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    for M in (int(a) for a in (sys.argv[1:] or ["256", "1024", "4096"])):
        x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda")
        ms = timeit(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y), 10)
        h = int(y.view(torch.int32).to(torch.int64).sum().item())
        print(f"{tag} K={K} N={N} M={M}: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s  bits={h:#x}", flush=True)
