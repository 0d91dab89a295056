"""Run one tcgen05 TBIK GEMM shape a few times (for ncu captures).
usage: prof_shape.py M K N [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

M, K, N = (int(a) for a in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, device="cuda")
cfg = tb.BlockConfig(64, 256, 128, 0)
for _ in range(reps):
    tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y)
torch.cuda.synchronize()
print("done", float(y[0, 0]))
