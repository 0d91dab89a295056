"""lm_head + log-softmax, two-pass vs the GEMM-epilogue chunk states (F2), device time
per call after an L2 flush.  usage: python tools/lm_head_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from tools.rowops_bench import ev_ms  # noqa: E402

cfg = tb.BlockConfig(64, 256, 128, 0)
for M, H, V, G in ((1024, 4096, 128256, 8), (4096, 4096, 128256, 8), (4096, 5120, 151936, 8), (512, 5120, 151936, 8)):
    g = torch.Generator(device="cuda")
    g.manual_seed(M)
    xa = (torch.randn(M, H, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    wl = (torch.randn(H, V, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    tg = torch.randint(0, V, (M,), device="cuda", generator=g)
    lg = torch.empty(M, V, device="cuda")
    ck = torch.empty(M, tb.chunk_states_per_row(V, G), 2, device="cuda")
    t_g = ev_ms(lambda: tb.tree_matmul(xa, wl, cfg, out=lg), 5)
    t_gf = ev_ms(lambda: tb.tree_matmul_logits(xa, wl, G, cfg, out=lg, chunks=ck), 5)
    for full in (False, True):
        t_u = ev_ms(lambda: (tb.tree_matmul(xa, wl, cfg, out=lg), tb.log_softmax(lg, G, 1, tg, full)), 5)
        t_f = ev_ms(lambda: (tb.tree_matmul_logits(xa, wl, G, cfg, out=lg, chunks=ck),
                             tb.log_softmax(lg, G, 1, tg, full, chunks=ck)), 5)
        print(f"M={M} H={H} V={V} full={full}: gemm {t_g:.3f} ms, gemm+chunk epilogue {t_gf:.3f} ms | "
              f"two-pass {t_u:.3f} ms, fused {t_f:.3f} ms", flush=True)
    del xa, wl, lg, ck
    torch.cuda.empty_cache()
