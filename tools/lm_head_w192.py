"""lm_head GEMM with and without the chunk (m, s) epilogue on the 256x128 / 256x192
kernels (device time per call, 20 back-to-back calls).  usage: lm_head_w192.py [M K V]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from tools.wide_check import ev_time  # noqa: E402

args = [int(a) for a in sys.argv[1:]]
M, K, V = args if len(args) == 3 else (1024, 4096, 128256)
G = 8
x = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
w = (torch.randn(K, V, device="cuda") * 0.02).to(torch.bfloat16)
cfg = tb.BlockConfig(64, 256, 128, 0)
lg = torch.empty(M, V, device="cuda")
ck = torch.empty(M, tb.chunk_states_per_row(V, G), 2, device="cuda")
tg = torch.randint(0, V, (M,), device="cuda")
for wv in (0, 1):
    with tb.schedule(tc_wide=wv):
        t = ev_time(lambda: tb.tree_matmul_logits(x, w, G, cfg, out=lg, chunks=ck))
        kern = tb.last_kernel()
        t2 = ev_time(lambda: tb.tree_matmul(x, w, cfg, out=lg))
        tf = ev_time(lambda: (tb.tree_matmul_logits(x, w, G, cfg, out=lg, chunks=ck),
                              tb.log_softmax(lg, G, 1, tg, False, chunks=ck)))
        tu = ev_time(lambda: (tb.tree_matmul(x, w, cfg, out=lg), tb.log_softmax(lg, G, 1, tg, False)))
        print(f"M={M} K={K} V={V} tc_wide={wv} ({kern}): GEMM+chunks {t:.1f} us, GEMM {t2:.1f} us | "
              f"fused lm_head+target log-probs {tf:.1f} us, two-pass {tu:.1f} us", flush=True)
