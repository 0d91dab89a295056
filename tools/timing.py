"""Shared timing helpers for the tools/ sweeps.

graph_time(fn, reps, rot): device microseconds per call of fn(i), measured as a
CUDA graph of `reps` calls rotating i over `rot` buffers (the host path -- Python +
C ABI, ~10 us -- would otherwise hide few-microsecond kernels).  The warm-up runs on
the capture stream itself: libtbik_b200's scratch arenas are per stream, so the
captured calls find theirs already sized (no allocation inside the capture).
"""
import torch


def graph_time(fn, reps=10, rot=3, replays=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(rot):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            fn(i % rot)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(replays):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (replays * reps)
