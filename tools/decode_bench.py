"""Decode-regime (small M) timing of the TBIK tree GEMM, Llama down_proj K=14336 N=4096:
  cold   one call after a 256 MB READ that evicts W from L2 (mean of 50; event quantum ~2 us)
  stream 40 back-to-back calls rotating over 4 weight copies (470 MB > L2): steady-state per call
usage: python tools/decode_bench.py [M ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

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
    for i in range(4):
        fn(i)
    torch.cuda.synchronize()
    s, e = ev(), ev()
    s.record()
    for i in range(reps):
        fn(i % 4)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps


def set_env(env):
    for k, v in env.items():
        os.environ[k] = v


for M in Ms:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    out = [f"M={M:4d}"]
    for name, env in (("wide", {"TBIK_TC_SKINNY": "0"}), ("skinny", {"TBIK_TC_SKINNY": "1"})):
        set_env(env)
        f = lambda i: tb.tree_matmul(x, ws[i], cfg, tb.LEAF_TCGEN05, out=y)  # noqa: E731
        c, st = cold(f), stream(f)
        out.append(f"{name} cold {c:5.1f} stream {st:5.1f} us ({K * N * 2 / st / 1e3:5.0f} GB/s)")
    os.environ.pop("TBIK_TC_SKINNY", None)
    f = lambda i: torch.matmul(x, ws[i], out=yb)  # noqa: E731
    c, st = cold(f), stream(f)
    out.append(f"cublas cold {c:5.1f} stream {st:5.1f} us ({K * N * 2 / st / 1e3:5.0f} GB/s)")
    print(" | ".join(out), flush=True)

# TP shard views (global k_first = 7): K/TP rows of the down_proj.  Device time per
# call from a CUDA graph of 20 calls (rotating 4 weight copies): the Python/C-ABI
# host path (~10 us per call) would otherwise hide these few-us kernels.


def graph_time(fn, reps=20):
    for i in range(4):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i % 4)
    g.replay()
    torch.cuda.synchronize()
    s, e = ev(), ev()
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / (5 * reps)


for tp in (1, 2, 4, 8):
    Ks = K // tp
    cfg_s = tb.BlockConfig(64, 256, 128, 7)
    for M in (1, 16, 64, 128):
        x = torch.randn(M, Ks, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda")
        wsh = [w[:Ks] for w in ws]
        out = [f"graph TP={tp} shard K={Ks:5d} M={M:3d}"]
        for name, env in (("wide", {"TBIK_TC_SKINNY": "0"}), ("skinny", {"TBIK_TC_SKINNY": "1"}),
                          ("sk_leaf", {"TBIK_TC_SKINNY": "1", "TBIK_SK_LEAF": "1"}),
                          ("sk_noleaf", {"TBIK_TC_SKINNY": "1", "TBIK_SK_LEAF": "0"}),
                          ("sk_u2", {"TBIK_TC_SKINNY": "1", "TBIK_SK_UNITS": "2", "TBIK_SK_LEAF": "0"}),
                          ("sk_u4", {"TBIK_TC_SKINNY": "1", "TBIK_SK_UNITS": "4", "TBIK_SK_LEAF": "0"}),
                          ("sk_bn64", {"TBIK_TC_SKINNY": "1", "TBIK_SK_BN": "64"}),
                          ("sk_bn128", {"TBIK_TC_SKINNY": "1", "TBIK_SK_BN": "128"})):
            set_env(env)
            f = lambda i: tb.tree_matmul(x, wsh[i], cfg_s, tb.LEAF_TCGEN05, out=y)  # noqa: E731
            st = graph_time(f)
            for k in env:
                os.environ.pop(k, None)
            out.append(f"{name} {st:5.1f}")
        yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        out.append(f"cublas {graph_time(lambda i: torch.matmul(x, wsh[i], out=yb)):5.1f} us")
        print(" | ".join(out), flush=True)
