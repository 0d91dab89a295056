"""A/B of programmatic dependent launch on the 256x192 kernel (knob tc_pdl): device
time per call over 20 back-to-back calls, and the bits.  usage: pdl_ab.py [M K N ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from tools.wide_check import ev_time  # noqa: E402

nums = [int(a) for a in sys.argv[1:] if a.isdigit()]
shapes = [tuple(nums[i:i + 3]) for i in range(0, len(nums), 3)] or [(4096, 14336, 4096), (1024, 4096, 28672),
                                                                    (4096, 4096, 4096), (2048, 14336, 4096),
                                                                    (1024, 4096, 4096), (1024, 14336, 4096),
                                                                    (512, 4096, 4096)]
for M, K, N in shapes:
    cfg = tb.BlockConfig(64, 256, 128, 0)
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    line, ref = [f"M={M} K={K} N={N}"], None
    for rep in range(2):
        for pdl in (0, 1):
            with tb.schedule(tc_pdl=pdl):
                t = ev_time(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y))
            same = True if ref is None else torch.equal(ref.view(torch.int32), y.view(torch.int32))
            if ref is None:
                ref = y.clone()
            line.append(f"pdl{pdl} {t:7.1f} us {2 * M * K * N / t / 1e6:6.0f} TF{'' if same else ' BITS DIFFER'}")
    print(" | ".join(line), flush=True)
