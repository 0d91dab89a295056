"""Time the deterministic GQA prefill attention kernels (tbik_attention_prefill, exact
two-pass order; tbik_attention_prefill_tc, tensor-core flash form) at
the Llama-3.1-8B forward shape (B=4, S=256, 32 q / 8 kv heads, D=128) against
PyTorch SDPA (non-deterministic-order, bf16 tensor cores)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from paper_2511_17826_b200._lib import check, lib  # noqa: E402

B, S, NQ, NKV, D = (int(a) for a in (sys.argv[1:] + ["4", "256", "32", "8", "128"][len(sys.argv) - 1:])[:5])
g = torch.Generator(device="cuda").manual_seed(3)
q = torch.randn(B * S, NQ * D, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(B * S, NKV * D, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(B * S, NKV * D, device="cuda", generator=g).to(torch.bfloat16)
o = torch.empty(B * S, NQ * D, device="cuda", dtype=torch.bfloat16)
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def run(fn=lib.tbik_attention_prefill):
    check(fn(C.c_void_p(q.data_ptr()), NQ * D, C.c_void_p(k.data_ptr()), NKV * D,
                                            C.c_void_p(v.data_ptr()), NKV * D, B, S, NQ, NKV, D, 1.0 / D ** 0.5,
                                            C.c_void_p(o.data_ptr()), NQ * D, st))


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


ms = timeit(run)
o1 = o.clone()
run()
same = torch.equal(o1.view(torch.int16), o.view(torch.int16))
qs, ks, vs = (t.view(B, S, -1, D).transpose(1, 2) for t in (q, k, v))
ms_sdpa = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qs, ks, vs, is_causal=True,
                                                                           enable_gqa=True))
fl = 4.0 * B * NQ * S * (S + 1) / 2 * D
ms_tc = timeit(lambda: run(lib.tbik_attention_prefill_tc))
print(f"tbik attention exact {ms*1e3:.1f} us ({fl/ms/1e9:.1f} TFLOP/s), run-to-run identical={same}; "
      f"tensor-core flash {ms_tc*1e3:.1f} us ({fl/ms_tc/1e9:.1f} TFLOP/s); SDPA {ms_sdpa*1e3:.1f} us")
