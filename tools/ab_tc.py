"""A/B: time tbik_tree_matmul from two builds of the library in one process."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_17826_b200 as tb  # noqa: E402
from paper_2511_17826_b200._lib import BlockConfigC  # noqa: E402


def bind(path):
    L = C.CDLL(path)
    L.tbik_tree_matmul.restype = C.c_int
    L.tbik_tree_matmul.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int, C.c_int64, C.c_void_p,
                                   C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.POINTER(BlockConfigC), C.c_int,
                                   C.c_void_p]
    return L


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    K, N = 14336, 4096
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    cfg = BlockConfigC(64, 256, 128, 0)
    libs = {"current": tb.lib, "v2": bind(os.path.join(ROOT, "tools", "ab", "libtbik_v2.so"))}
    outs = {}
    for rnd in range(2):
        for name, L in libs.items():
            s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
            call = lambda: L.tbik_tree_matmul(x.data_ptr(), 1, K, w.data_ptr(), 1, N, y.data_ptr(), N, M, N, K,
                                              C.byref(cfg), 1, s)
            for _ in range(3):
                assert call() == 0
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                call()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 20
            outs[name] = y.clone()
            print(f"round {rnd} {name:8s} M={M}: {ms*1e3:7.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s", flush=True)
    print("bits equal:", torch.equal(outs["current"].view(torch.int32), outs["v2"].view(torch.int32)))


if __name__ == "__main__":
    main()
