"""Small-M tuning of the tcgen05 TBIK GEMM: A rows per stage (TBIK_TC_ABOX) x K split
(TBIK_TC_UNITS) at the Llama down_proj shape, each timed with an L2 flush before
every call (W = 117 MB would otherwise sit in the 126 MB L2; the flush READS 256 MB
so no dirty lines are left to be written back during the timed call).  Every configuration
must give identical bits."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17826_b200 as tb  # noqa: E402

K = int(os.environ.get("K", 14336))
N = int(os.environ.get("N", 4096))
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB, READ to evict (no dirty lines)
sink = torch.empty((), device="cuda")


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        torch.sum(flush, dim=0, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
cfg = tb.BlockConfig(64, 256, 128, 0)
for M in (int(a) for a in (sys.argv[1:] or ["1", "16", "32", "64", "128", "256"])):
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    ref = None
    for pair in ("0", "1"):
        if pair == "0" and M > int(os.environ.get("TUNE_SINGLE_MAX_M", "128")):
            continue
        for abox in ("32", "64", "128"):
            if int(abox) < M and abox != "128":
                continue
            for u in ("1", "2", "4"):
                os.environ["TBIK_TC_PAIR"] = pair
                os.environ["TBIK_TC_ABOX"] = abox
                os.environ["TBIK_TC_UNITS"] = u
                ms = timed(lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y))
                ref = y.clone() if ref is None else ref
                same = torch.equal(ref.view(torch.int32), y.view(torch.int32))
                print(f"M={M} pair={pair} abox={abox} units={u}: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s "
                      f"W-stream {2*K*N/ms/1e6:6.0f} GB/s bits_equal={same}", flush=True)
    os.environ.pop("TBIK_TC_PAIR")
    os.environ.pop("TBIK_TC_UNITS")
    os.environ.pop("TBIK_TC_ABOX")
    yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ms = timed(lambda: torch.matmul(x, w, out=yb))
    print(f"M={M} cuBLAS: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s W-stream {2*K*N/ms/1e6:6.0f} GB/s",
          flush=True)
