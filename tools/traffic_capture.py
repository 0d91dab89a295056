"""DRAM traffic per launch of every kernel the bench line reports a roofline for, for
`profiles/ncu_traffic.json`.  Run under
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
      --clock-control none -k regex:tbik_b200 --csv --log-file OUT python tools/traffic_capture.py
(ncu flushes the caches before every kernel: cold-cache bytes).  Each step runs its
entry point ONCE and prints `step <name> <launches>` so tools/traffic_reduce.py can
attribute the kernel rows in order."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_17826_b200 as tb  # noqa: E402


def step(name, fn):
    torch.cuda.synchronize()
    n0 = tb.launch_count()
    fn()
    torch.cuda.synchronize()
    print(f"step {name} {tb.launch_count() - n0}", flush=True)


def main():
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    M, K, N = 4096, 14336, 4096
    x = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    w = torch.randn(K, N, device=dev, generator=g).to(torch.bfloat16)
    y = torch.empty(M, N, device=dev)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    step("M4096_tp1", lambda: tb.tree_matmul(x, w, cfg, tb.LEAF_TCGEN05, out=y))
    kf = tb.plan_blocks(K, cfg, 8).k_first
    for t in (2, 4, 8):
        sp = tb.make_row_shard_plan(K, cfg, t, 8)
        kb, ke = sp.bounds[0]
        xs, ws = x[:, kb:ke].contiguous(), w[kb:ke].contiguous()
        cfg_t = tb.BlockConfig(64, 256, 128, kf)
        step(f"M4096_shard_tp{t}", lambda: tb.tree_matmul(xs, ws, cfg_t, tb.LEAF_TCGEN05, out=y))
        del xs, ws
    del x, w, y
    torch.cuda.empty_cache()

    H, V, groups = 5120, 151936, 8
    xr = torch.randn(M, H, device=dev, generator=g).to(torch.bfloat16)
    gamma = 1 + 0.02 * torch.randn(H, device=dev, generator=g)
    step("rmsnorm_bf16", lambda: tb.rmsnorm(xr, gamma, 1e-6, out_dtype=torch.bfloat16))
    del xr
    logits = torch.randn(M, V, device=dev, generator=g) * 4.0
    targets = torch.randint(0, V, (M,), device=dev, generator=g)
    for tp in (1, 8):
        step(f"log_softmax_full_tp{tp}", lambda: tb.log_softmax(logits, groups, tp, None, True))
        step(f"log_softmax_targets_tp{tp}", lambda: tb.log_softmax(logits, groups, tp, targets, False))
    del logits
    torch.cuda.empty_cache()
    E = M * 4096
    for W in (2, 4, 8):
        parts = [torch.randn(E, device=dev, generator=g) for _ in range(W)]
        grp = tb.DeviceGroup(W)
        step(f"allreduce_W{W}", lambda: tb.tree_all_reduce(grp, parts))
        del parts


if __name__ == "__main__":
    main()
