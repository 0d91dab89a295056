"""One TP-shard decode GEMM (default: the Llama down_proj TP = 8 shard, M=16 K=1792
N=4096, k_first = 7 -- one leaf group) through the TBIK skinny kernel and cuBLAS, a
few times each, for ncu captures.  usage: prof_decode.py [M K N kf reps] [--knob k=v ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

knobs = {}
argv = sys.argv[1:]
for i, a in enumerate(argv):
    if a == "--knob":
        k, v = argv[i + 1].split("=")
        knobs[k] = int(v)
nums = [int(a) for i, a in enumerate(argv) if a.isdigit() and (i == 0 or argv[i - 1] != "--knob")]
M, K, N, kf, reps = (nums + [16, 1792, 4096, 7, 3][len(nums):])[:5]
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, device="cuda")
cfg = tb.BlockConfig(64, 256, 128, kf)
with tb.schedule(**knobs):
    for _ in range(reps):
        tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y)
yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    torch.matmul(x, w, out=yb)
torch.cuda.synchronize()
print("done", float(y[0, 0]))
