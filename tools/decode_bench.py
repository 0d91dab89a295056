"""Decode-regime (small M) timing of the TBIK tree GEMM, Llama down_proj K=14336 N=4096:
  cold   one call after a 256 MB READ that evicts W from L2 (mean of 50; event quantum ~2 us)
  stream 40 back-to-back calls rotating over 4 weight copies (470 MB > L2): steady-state per call
usage: python tools/decode_bench.py [M ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402
from tools.timing import graph_time  # noqa: E402

K, N = 14336, 4096
cfg = tb.BlockConfig(64, 256, 128, 0)
Ms = [int(a) for a in sys.argv[1:] if a.isdigit()] or [1, 4, 8, 16, 32, 64, 128]
ws = [torch.randn(K, N, device="cuda").to(torch.bfloat16) for _ in range(4)]
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")


def ev():
    return torch.cuda.Event(enable_timing=True)


def cold(fn, reps=50):
    tot = 0.0
    for _ in range(reps):
        torch.sum(flush, dim=0, out=sink)
        s, e = ev(), ev()
        s.record()
        fn(0)
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e) * 1e3
    return tot / reps


def stream(fn, reps=40):
    return graph_time(fn, reps=reps, rot=4)


def graph_time_20(fn):
    return graph_time(fn, reps=20, rot=4)


for M in Ms:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    out = [f"M={M:4d}"]
    for name, knobs in (("wide", {"tc_skinny": 0}), ("skinny", {"tc_skinny": 1}),
                        ("skinny ks64", {"tc_skinny": 1, "sk_ks": 64}),
                        ("skinny nopdl", {"tc_skinny": 1, "sk_pdl": 0})):
        f = lambda i: tb.tree_matmul(x, ws[i], cfg, tb.LEAF_TCGEN05, out=y)  # noqa: E731
        with tb.schedule(**knobs):
            c, st = cold(f), stream(f)
        out.append(f"{name} cold {c:5.1f} stream {st:5.1f} us ({K * N * 2 / st / 1e3:5.0f} GB/s)")
    f = lambda i: torch.matmul(x, ws[i], out=yb)  # noqa: E731
    c, st = cold(f), stream(f)
    out.append(f"cublas cold {c:5.1f} stream {st:5.1f} us ({K * N * 2 / st / 1e3:5.0f} GB/s)")
    print(" | ".join(out), flush=True)

# TP shard views (global k_first = 7): K/TP rows of the down_proj.  Device time per
# call from a CUDA graph of 20 calls (rotating 4 weight copies): the Python/C-ABI
# host path (~10 us per call) would otherwise hide these few-us kernels.


for tp in (1, 2, 4, 8):
    Ks = K // tp
    cfg_s = tb.BlockConfig(64, 256, 128, 7)
    for M in (1, 16, 64, 128):
        x = torch.randn(M, Ks, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda")
        wsh = [w[:Ks] for w in ws]
        out = [f"graph TP={tp} shard K={Ks:5d} M={M:3d}"]
        for name, knobs in (("wide", {"tc_skinny": 0}), ("skinny", {"tc_skinny": 1}),
                            ("sk_leaf", {"tc_skinny": 1, "sk_leaf": 1}),
                            ("sk_noleaf", {"tc_skinny": 1, "sk_leaf": 0}),
                            ("sk_u2", {"tc_skinny": 1, "sk_units": 2, "sk_leaf": 0}),
                            ("sk_u4", {"tc_skinny": 1, "sk_units": 4, "sk_leaf": 0}),
                            ("sk_bn32", {"tc_skinny": 1, "sk_bn": 32}),
                            ("sk_bn64", {"tc_skinny": 1, "sk_bn": 64}),
                            ("sk_bn128", {"tc_skinny": 1, "sk_bn": 128}),
                            ("sk_ks64", {"tc_skinny": 1, "sk_ks": 64}),
                            ("sk_bn64_ks64", {"tc_skinny": 1, "sk_bn": 64, "sk_ks": 64}),
                            ("sk_bn128_ks64", {"tc_skinny": 1, "sk_bn": 128, "sk_ks": 64}),
                            ("sk_nopdl", {"tc_skinny": 1, "sk_pdl": 0}),
                            ("sk_nopair", {"tc_skinny": 1, "sk_pair": 0})):
            f = lambda i: tb.tree_matmul(x, wsh[i], cfg_s, tb.LEAF_TCGEN05, out=y)  # noqa: E731
            with tb.schedule(**knobs):
                st = graph_time_20(f)
            out.append(f"{name} {st:5.1f}")
        yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        out.append(f"cublas {graph_time_20(lambda i: torch.matmul(x, wsh[i], out=yb)):5.1f} us")
        print(" | ".join(out), flush=True)
