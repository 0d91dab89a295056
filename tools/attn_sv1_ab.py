import os, sys, torch, ctypes as C
sys.path.insert(0, os.getcwd())
import paper_2511_17826_b200 as tb
from paper_2511_17826_b200._lib import lib
from tools.wide_check import ev_time
D = 128
for B, S, nq, nkv in [(4, 256, 32, 8), (1, 512, 64, 8), (8, 128, 32, 8), (2, 512, 32, 8)]:
    q = torch.randn(B * S, nq * D, device="cuda").to(torch.bfloat16)
    k = torch.randn(B * S, nkv * D, device="cuda").to(torch.bfloat16)
    v = torch.randn(B * S, nkv * D, device="cuda").to(torch.bfloat16)
    o = torch.empty(B * S, nq * D, device="cuda", dtype=torch.bfloat16)
    vp = lambda t: C.c_void_p(t.data_ptr())
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    line = [f"B={B} S={S} nq={nq}"]
    for rep in range(2):
        for sv1 in (0, 1):
            with tb.schedule(attn_sv1=sv1):
                t = ev_time(lambda: lib.tbik_attention_prefill_tc(vp(q), nq * D, vp(k), nkv * D, vp(v), nkv * D, B, S, nq, nkv, D, 0.088, vp(o), nq * D, st))
            line.append(f"sv1={sv1} {t:6.1f} us")
    print(" | ".join(line), flush=True)
