"""Small launches of the 256x192 / 256x128 tree GEMMs (ragged M/N/K, scratch levels,
half items, SiLU epilogue) for compute-sanitizer runs.  usage: compute-sanitizer
--tool memcheck python tools/sanitize_w192.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(1)
for M, K, N, bk, kf in [(300, 3000, 520, 256, 0), (777, 4096, 200, 256, 1), (513, 8192, 97, 128, 0),
                        (2300, 1000, 1000, 64, 0)]:
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
    cfg = tb.BlockConfig(64, bk, 128, kf)
    outs = []
    for wv in (0, 1):
        with tb.schedule(tc_wide=wv):
            outs.append(tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05))
    torch.cuda.synchronize()
    print(M, K, N, "same" if torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32)) else "DIFFER",
          flush=True)
x = torch.randn(600, 4096, device="cuda", generator=g).to(torch.bfloat16)
w = (torch.randn(4096, 2 * 1000, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
with tb.schedule(tc_wide=1):
    a = tb.tree_matmul_silu_mul(x, tb.interleave_gate_up(w), tb.DeviceGroup(1), tb.BlockConfig(64, 256, 128, 0))
torch.cuda.synchronize()
print("silu ok", tb.last_kernel())
