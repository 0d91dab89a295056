"""One C5-sized tree RMSNorm (4096 x 5120 bf16 -> bf16) a few times, for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

x = torch.randn(4096, 5120, device="cuda").to(torch.bfloat16)
gamma = 1 + 0.02 * torch.randn(5120, device="cuda")
for _ in range(3):
    tb.rmsnorm(x, gamma, 1e-6, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
print("done")
