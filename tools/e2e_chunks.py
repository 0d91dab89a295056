"""Sweep the host-io chunk size of tbik_tree_matmul_hostio at the bench shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

M, K, N = 4096, 14336, 4096
x = torch.randn(M, K).to(torch.bfloat16).pin_memory()
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N).pin_memory()
cfg = tb.BlockConfig(64, 256, 128, 0)
xd = x.cuda()
for chunk in (0, 256, 384, 512, 1024, 4096):
    for _ in range(2):
        tb.tree_matmul_hostio(x, w, cfg, tb.LEAF_TCGEN05, out=y, chunk_rows=chunk)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        tb.tree_matmul_hostio(x, w, cfg, tb.LEAF_TCGEN05, out=y, chunk_rows=chunk)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"chunk={chunk}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.1f} TFLOP/s", flush=True)
for name, fn in (("h2d only", lambda: xd.copy_(x, non_blocking=True)),
                 ("d2h only", lambda: y.copy_(torch.empty(M, N, device="cuda"), non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(name, a.elapsed_time(b) / 5, "ms")
