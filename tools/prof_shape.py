"""Run one TBIK GEMM shape (and optionally the cuBLAS bf16 GEMM of the same shape)
a few times, for ncu captures.
usage: prof_shape.py M K N [reps] [--cublas] [--knob name=value ...]"""
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
argv = [a for i, a in enumerate(argv) if a != "--knob" and (i == 0 or argv[i - 1] != "--knob")]
args = [a for a in argv if not a.startswith("--")]
M, K, N = (int(a) for a in args[:3])
reps = int(args[3]) if len(args) > 3 else 3
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, device="cuda")
cfg = tb.BlockConfig(64, 256, 128, 0)
with tb.schedule(**knobs):
    for _ in range(reps):
        tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y)
if "--cublas" in sys.argv:
    yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(reps):
        torch.matmul(x, w, out=yb)
torch.cuda.synchronize()
print("done", float(y[0, 0]))
