"""Kernel-time breakdown of the TBIK decoder forward (torch.profiler / CUPTI sees
every kernel, including the C-ABI ones).  usage: fwd_profile.py [layers] [batch] [seq]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_17826_b200 import model as mdl  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 4
seq = int(sys.argv[3]) if len(sys.argv) > 3 else 256
cfg = mdl.llama31_8b()
cfg.n_layers = layers
w = mdl.random_weights(cfg, seed=3)
dec = mdl.TbikDecoder(cfg, w)
tokens = torch.randint(0, cfg.vocab, (batch, seq), device="cuda")


def step():
    logits = dec.forward(tokens, 1)
    return dec.log_probs(logits, 1, full=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
