"""The Llama-3.1-8B prefill attention (4 x 256 tokens, 32 q / 8 kv heads) a few times, for ncu.
usage: prof_attn.py [attn_tc5 knob (default 0)] [B S]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402,F401
from paper_2511_17826_b200._lib import lib  # noqa: E402

nums = [int(a) for a in sys.argv[1:]]
tc5 = nums[0] if nums else 0
B, S = (nums[1], nums[2]) if len(nums) >= 3 else (4, 256)
nq, nkv, D = 32, 8, 128
q = torch.randn(B * S, nq * D, device="cuda").to(torch.bfloat16)
k = torch.randn(B * S, nkv * D, device="cuda").to(torch.bfloat16)
v = torch.randn(B * S, nkv * D, device="cuda").to(torch.bfloat16)
o = torch.empty(B * S, nq * D, device="cuda", dtype=torch.bfloat16)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    tb.set_schedule("attn_tc5", tc5)
    lib.tbik_attention_prefill_tc(vp(q), nq * D, vp(k), nkv * D, vp(v), nkv * D, B, S, nq, nkv, D, 0.088, vp(o),
                                  nq * D, st)
torch.cuda.synchronize()
print("done")
