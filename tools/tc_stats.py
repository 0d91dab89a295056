"""Per-role wait-cycle breakdown of the tcgen05 TBIK GEMM (TBIK_TC_STATS=1)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["TBIK_TC_STATS"] = "1"
import paper_2511_17826_b200 as tb  # noqa: E402

tb.lib.tbik_debug_tc_stats.restype = C.c_int
tb.lib.tbik_debug_tc_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]


def run(M, K, N, bn):
    os.environ["TBIK_TC_BN"] = str(bn)
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    for _ in range(3):
        tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05)
    buf = (C.c_ulonglong * 4096)()
    n = tb.lib.tbik_debug_tc_stats(buf, 4096)
    rows = [[buf[i * 8 + j] for j in range(8)] for i in range(n // 8)]
    lead = rows[0::2]
    avg = lambda col, rs: sum(r[col] for r in rs) / len(rs)
    loop = avg(4, rows)
    print(f"M={M} K={K} N={N} BN={bn}: ctas={len(rows)} producer_loop={loop:.0f} cyc | "
          f"producer empty-wait {avg(0, rows)/loop:.1%} | MMA tempty-wait {avg(1, lead)/loop:.1%} | "
          f"MMA full-wait {avg(2, lead)/loop:.1%} | merge tfull-wait {avg(3, rows)/avg(5, rows):.1%} | "
          f"merge busy {avg(6, rows)/avg(5, rows):.1%}", flush=True)


if __name__ == "__main__":
    for bn in (128, 256):
        run(4096, 14336, 4096, bn)
        run(1024, 14336, 4096, bn)
