"""A/B of the attention kernel's output bits between two builds of the library
(argv[1], argv[2]) through the C ABI: prints whether the outputs are identical."""
import ctypes as C
import sys

import torch

B, S, nq, nkv, D = 3, 1000, 8, 2, 128
g = torch.Generator(device="cuda").manual_seed(11)
q = (torch.randn(B * S, nq * D, device="cuda", generator=g) * 2).to(torch.bfloat16)
k = (torch.randn(B * S, nkv * D, device="cuda", generator=g) * 2).to(torch.bfloat16)
v = torch.randn(B * S, nkv * D, device="cuda", generator=g).to(torch.bfloat16)
outs = []
for path in sys.argv[1:3]:
    lib = C.CDLL(path)
    o = torch.empty(B * S, nq * D, device="cuda", dtype=torch.bfloat16)
    f = lib.tbik_attention_prefill_tc
    f.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int,
                  C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_int64, C.c_void_p]
    st = f(q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0), v.data_ptr(), v.stride(0), B, S, nq, nkv, D,
           D ** -0.5, o.data_ptr(), o.stride(0), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert st == 0, st
    outs.append(o)
print("attention bits identical between builds:", torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16)))
