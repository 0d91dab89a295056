"""Small launches of the skinny (decode) tree GEMM in every mode -- persistent single
unit, in-cluster K-split finish, CTA-pair handoffs (leaf split / two subtree units),
32/64/128-column tiles, 64/128-row stages, PDL -- for compute-sanitizer runs.
usage: compute-sanitizer --tool memcheck python tools/sanitize_skinny.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(2)
cases = [  # M, K, N, k_first, knobs
    (16, 1792, 1000, 7, {}),                      # pair mode 1 (leaf split)
    (5, 3584, 700, 7, {}),                        # pair mode 2 (two subtree units)
    (64, 1792, 512, 7, {}),                       # pair mode 1, 64 tokens
    (33, 7168, 384, 7, {}),                       # cluster finish (4 units)
    (128, 2048, 300, 0, {}),                      # 128 tokens
    (16, 1792, 333, 7, {"sk_pair": 0}),           # single CTA per tile
    (16, 1792, 640, 7, {"sk_bn": 32}),            # 32-column tiles
    (16, 1792, 640, 7, {"sk_ks": 64}),            # 64-row stages
    (16, 777, 640, 4, {}),                        # partial last leaf
    (16, 4096, 20000, 0, {"sk_units": 1}),        # persistent CTAs over several tiles
]
for M, K, N, kf, knobs in cases:
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, kf)
    with tb.schedule(tc_skinny=0):
        ref = tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05)
    with tb.schedule(tc_skinny=1, **knobs):
        y = tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05)
        y2 = tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05)  # back to back (PDL)
    torch.cuda.synchronize()
    same = torch.equal(y.view(torch.int32), ref.view(torch.int32)) and torch.equal(y2.view(torch.int32),
                                                                                      ref.view(torch.int32))
    print(M, K, N, kf, knobs, tb.last_kernel(), "same" if same else "DIFFER", flush=True)
