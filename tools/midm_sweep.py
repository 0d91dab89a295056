"""Mid-M schedule sweep of the wide tcgen05 kernel (pure scheduling knobs, same bits):
Llama down_proj K=14336 N=4096 and o_proj K=4096 N=4096 at M = 256..2048; device time
per call from a CUDA graph of 10 calls rotating 3 weight copies.
usage: python tools/midm_sweep.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

cfg = tb.BlockConfig(64, 256, 128, 0)
KNOBS = ("TBIK_TC_WIDE", "TBIK_TC_UNITS", "TBIK_TC_DEEP", "TBIK_TC_GROUP_M", "TBIK_TC_SKINNY", "TBIK_TC_EPI",
         "TBIK_TC_MC")
VARIANTS = [("default", {}), ("wide", {"TBIK_TC_WIDE": "1"}), ("units2", {"TBIK_TC_UNITS": "2"}),
            ("units4", {"TBIK_TC_UNITS": "4"}), ("deep0", {"TBIK_TC_DEEP": "0"}), ("deep1", {"TBIK_TC_DEEP": "1"}),
            ("gm4", {"TBIK_TC_GROUP_M": "4"}), ("epi16", {"TBIK_TC_EPI": "16"})]
if "--epi" in sys.argv:
    VARIANTS = [("default", {}), ("epi16", {"TBIK_TC_EPI": "16"})]
if "--mc" in sys.argv:
    VARIANTS = [("default", {}), ("mc", {"TBIK_TC_MC": "1"}), ("mc_u1", {"TBIK_TC_MC": "1", "TBIK_TC_UNITS": "1"}),
                ("mc_u2", {"TBIK_TC_MC": "1", "TBIK_TC_UNITS": "2"}), ("units1", {"TBIK_TC_UNITS": "1"})]


def graph_time(fn, reps=10):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i % 3)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / (5 * reps)


for K, N in ((14336, 4096), (4096, 4096), (4096, 28672)):
    ws = [torch.randn(K, N, device="cuda").to(torch.bfloat16) for _ in range(3)]
    for M in ((1024, 2048, 4096) if "--epi" in sys.argv else (256, 512, 768, 1024, 1536, 2048)):
        if "--mc" in sys.argv and M > 1024:
            continue
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda")
        ref = None
        line = [f"K={K} N={N} M={M:5d}"]
        for name, env in VARIANTS:
            for k in KNOBS:
                os.environ.pop(k, None)
            os.environ.update(env)
            f = lambda i: tb.tree_matmul(x, ws[i], cfg, tb.LEAF_TCGEN05, out=y)  # noqa: E731
            t = graph_time(f)
            if ref is None:
                ref = y.clone()
            same = torch.equal(ref.view(torch.int32), y.view(torch.int32))
            line.append(f"{name} {2 * M * K * N / t / 1e6:6.0f}{'' if same else '!'}")
        for k in KNOBS:
            os.environ.pop(k, None)
        yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t = graph_time(lambda i: torch.matmul(x, ws[i], out=yb))
        line.append(f"cublas {2 * M * K * N / t / 1e6:6.0f} TFLOP/s")
        print(" | ".join(line), flush=True)
