"""One TBIK forward (for ncu launch lists): python tools/forward_once.py [layers] [batch] [seq]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_17826_b200 import model as mdl  # noqa: E402

layers, batch, seq = (int(a) for a in (sys.argv[1:] + ["4", "4", "256"][len(sys.argv) - 1:])[:3])
cfg = mdl.llama31_8b(layers)
w = mdl.random_weights(cfg, seed=3)
dec = mdl.TbikDecoder(cfg, w)
tokens = torch.randint(0, cfg.vocab, (batch, seq), device="cuda")
for _ in range(2):
    logits = dec.forward(tokens, 1)
    dec.log_probs(logits, 1)
torch.cuda.synchronize()
