import torch, sys
sys.path.insert(0, ".")
import paper_2511_17826_b200 as tb
from tools.wide_check import ev_time
for (M, K, N) in [(1024, 4096, 4096), (768, 4096, 4096), (512, 4096, 4096), (1024, 14336, 4096)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    cfg = tb.BlockConfig(64, 256, 128, 0)
    line = [f"M={M} K={K} N={N}"]
    for name, kn in [("auto", {}), ("n_u1", {"tc_wide": 0, "tc_units": 1}), ("n_u2", {"tc_wide": 0, "tc_units": 2}), ("n_u4", {"tc_wide": 0, "tc_units": 4}), ("n_u8", {"tc_wide": 0, "tc_units": 8}), ("w_u2", {"tc_wide": 1, "tc_units": 2}), ("w_u4", {"tc_wide": 1, "tc_units": 4})]:
        with tb.schedule(**kn):
            t = ev_time(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y))
        line.append(f"{name} {t:.1f}")
    yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    line.append(f"cublas {ev_time(lambda: torch.matmul(x, w, out=yb)):.1f}")
    print(" | ".join(line), flush=True)
