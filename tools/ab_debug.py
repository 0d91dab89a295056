"""Where the tc GEMM's time goes at k_first = 1 vs 7: TBIK_TC_DEBUG ablations (WRONG results,
timing only): 1 = skip the merge, 2 = skip the output store, 4 = skip the tree above level 0.
TBIK_TC_DEBUG is read once per process, so each variant runs in its own process.
usage: python tools/ab_debug.py  (driver)   |   python tools/ab_debug.py run K N M"""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2511_17826_b200 as tb
    K, N, M = (int(a) for a in sys.argv[2:5])
    cfg = tb.BlockConfig(64, 256, 128, 0)
    ws = [torch.randn(K, N, device="cuda").to(torch.bfloat16) for _ in range(3)]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    for i in range(3):
        tb.tree_matmul(x, ws[i], cfg, tb.LEAF_TCGEN05, out=y)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(10):
            tb.tree_matmul(x, ws[i % 3], cfg, tb.LEAF_TCGEN05, out=y)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) * 1e3 / 50
    print(f"{2 * M * K * N / t / 1e6:.0f}")
    sys.exit(0)

SHAPES = ((4096, 4096, 2048), (4096, 4096, 4096), (14336, 4096, 4096), (4096, 28672, 1024))
DBG = ("0", "1", "2", "4", "6")
if "--store" in sys.argv:  # TMA-store output staging vs direct row stores (debug 16)
    SHAPES = ((4096, 4096, 4096), (1792, 4096, 4096), (14336, 4096, 4096), (4096, 28672, 1024))
    DBG = ("0", "16", "2")
for K, N, M in SHAPES:
    line = [f"K={K} N={N} M={M}"]
    for dbg in DBG:
        env = dict(os.environ, TBIK_TC_DEBUG=dbg)
        out = subprocess.run([sys.executable, __file__, "run", str(K), str(N), str(M)], env=env,
                             capture_output=True, text=True).stdout.strip()
        line.append(f"debug={dbg}: {out}")
    print(" | ".join(line), flush=True)
