"""BASELINE configs[4] on one B200: tree RMSNorm + vocab-sharded tree log-softmax
(4096 tokens, Qwen3-32B hidden 5120, vocab 151936), and the fixed-order tree
all-reduce of the row-parallel partials.  All three are HBM-bound; each call is
timed alone with CUDA events after an L2 eviction (a 256 MB read: the RMSNorm
working set fits the 126 MB L2) and reported as algorithmic GB/s against
MEASURED_PEAKS.json hbm_gbs.  Prints one JSON object (also imported by
bench.py).

Algorithmic bytes:
  rmsnorm       read 2*M*H (bf16) + 4*H (gamma), write 2*M*H (bf16 out)
  log-softmax   pass 1 (m, s) leaves: read 4*M*V ; finish: read 4*M*V + write 4*M*V
                (full log-prob matrix) or read 4*M + 4*M (target log-probs only)
  all-reduce    read 4*W*E (W partials) + write 4*E
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_17826_b200 as tb  # noqa: E402


_FLUSH = None


def ev_ms(fn, reps=20):
    """Device time (ms) per call, every call preceded by a 256 MB read that evicts
    the 126 MB L2 (the RMSNorm working set, 84 MB, would otherwise stay resident
    between reps); only fn is inside the events."""
    global _FLUSH
    if _FLUSH is None:
        _FLUSH = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    sink = torch.empty((), device="cuda")
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        torch.sum(_FLUSH, dim=0, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


_TRAFFIC = None


def traffic(key):
    """Cold-cache DRAM bytes (read + write) per call from the committed ncu capture
    (profiles/ncu_traffic.json, tools/traffic_capture.py), or None."""
    global _TRAFFIC
    if _TRAFFIC is None:
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                _TRAFFIC = json.load(f)
        except Exception:  # noqa: BLE001
            _TRAFFIC = {}
    return _TRAFFIC.get(key)


def line(name, nbytes, ms, peak, key=None):
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"kernel": name, "ms": ms, "alg_bytes": nbytes, "GB/s": gbs, "frac_of_hbm": gbs / peak,
            "traffic": traffic(key) if key else None}


def run(M=4096, H=5120, V=151936, groups=8, tps=(1, 2, 4, 8), reps=20):
    dev = torch.device("cuda")
    peak, src = hbm_peak()
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    out = {"config": {"tokens": M, "hidden": H, "vocab": V, "vocab_groups": groups},
           "hbm_peak_gbs": peak, "peak_source": src}

    # ---- tree RMSNorm (bf16 in, bf16 out; and f32 in -> f32 out) -----------------------
    x = torch.randn(M, H, device=dev, generator=g).to(torch.bfloat16)
    gamma = (1 + 0.02 * torch.randn(H, device=dev, generator=g))
    ms = ev_ms(lambda: tb.rmsnorm(x, gamma, 1e-6, out_dtype=torch.bfloat16), reps)
    out["rmsnorm_bf16"] = line("tree_rmsnorm_kernel (bf16->bf16)", 4.0 * M * H + 4 * H, ms, peak, "rmsnorm_bf16")
    ms_t = ev_ms(lambda: (x.float() * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-6)
                          * gamma).to(torch.bfloat16), reps)
    out["rmsnorm_bf16"]["torch_eager_ms"] = ms_t
    # replicated across ranks -> TP-invariant; batch invariance: row 0 alone equals row 0 in the batch
    y_all = tb.rmsnorm(x, gamma, 1e-6, out_dtype=torch.bfloat16)
    y_one = tb.rmsnorm(x[:1].contiguous(), gamma, 1e-6, out_dtype=torch.bfloat16)
    out["rmsnorm_bf16"]["batch_invariant"] = bool(torch.equal(y_all[:1].view(torch.int16), y_one.view(torch.int16)))
    del x, y_all, y_one

    # ---- vocab-sharded tree log-softmax --------------------------------------------------
    logits = torch.randn(M, V, device=dev, generator=g) * 4.0
    targets = torch.randint(0, V, (M,), device=dev, generator=g)
    full_bytes = 4.0 * M * V * 3            # (m, s) pass + finish read + log-prob write
    tgt_bytes = 4.0 * M * V + 16.0 * M      # (m, s) pass + per-row target gather + writes
    res = {}
    ref = None
    for tp in tps:
        ms_full = ev_ms(lambda: tb.log_softmax(logits, groups, tp, None, True), reps)
        ms_tgt = ev_ms(lambda: tb.log_softmax(logits, groups, tp, targets, False), reps)
        lse, lp, _ = tb.log_softmax(logits, groups, tp, None, True)
        _, _, tlp = tb.log_softmax(logits, groups, tp, targets, False)
        if ref is None:
            ref = (lse.clone(), lp.clone(), tlp.clone())
            same = True
        else:
            same = (torch.equal(ref[0].view(torch.int32), lse.view(torch.int32))
                    and torch.equal(ref[1].view(torch.int32), lp.view(torch.int32))
                    and torch.equal(ref[2].view(torch.int32), tlp.view(torch.int32)))
        res[f"tp{tp}"] = {"full": line("log-softmax full (ms_group + merge + finish)", full_bytes, ms_full, peak,
                                       f"log_softmax_full_tp{tp}"),
                          "target_logprobs": line("log-prob of targets", tgt_bytes, ms_tgt, peak,
                                                  f"log_softmax_targets_tp{tp}"),
                          "bit_identical_to_tp1": bool(same)}
        del lse, lp, tlp
    ms_t = ev_ms(lambda: torch.log_softmax(logits, -1), reps)
    res["torch_log_softmax_ms"] = ms_t
    ref_lp = torch.log_softmax(logits.double(), -1)
    res["max_abs_err_vs_f64"] = float((ref[1].double() - ref_lp).abs().max())
    out["log_softmax"] = res
    del ref, ref_lp
    torch.cuda.empty_cache()

    # ---- F2: lm_head + log-softmax, unfused vs the epilogue-fused chunk states -----------
    # (M tokens x hidden H) . (H x V) bf16 lm_head, then lse + target log-probs: unfused =
    # tree GEMM, then the log-softmax reads the 4 M V logits again; fused = the GEMM's
    # epilogue writes the 16-logit (m, s) chunk states (0.5 B per logit) and the first
    # pass reads those instead.  Same bits (tested).
    del logits
    torch.cuda.empty_cache()
    xa = (torch.randn(M, H, device=dev, generator=g) * 0.5).to(torch.bfloat16)
    wl = (torch.randn(H, V, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    cfg = tb.BlockConfig(64, 256, 128, 0)
    lg = torch.empty(M, V, device=dev)

    def unfused():
        tb.tree_matmul(xa, wl, cfg, out=lg)
        tb.log_softmax(lg, groups, 1, targets, False)

    ck = torch.empty(M, tb.chunk_states_per_row(V, groups), 2, device=dev)

    def fused():
        tb.tree_matmul_logits(xa, wl, groups, cfg, out=lg, chunks=ck)
        tb.log_softmax(lg, groups, 1, targets, False, chunks=ck)

    ms_u = ev_ms(unfused, max(reps // 4, 3))
    ms_f = ev_ms(fused, max(reps // 4, 3))
    ms_g = ev_ms(lambda: tb.tree_matmul(xa, wl, cfg, out=lg), max(reps // 4, 3))
    out["lm_head_logsoftmax"] = {"M": M, "H": H, "V": V, "gemm_ms": ms_g, "unfused_ms": ms_u, "fused_ms": ms_f,
                                 "saved_ms": ms_u - ms_f,
                                 "path": "tree_matmul + log_softmax(logits) vs tree_matmul_logits + "
                                         "log_softmax(chunk states); target log-probs, L2 flushed before each call"}
    del xa, wl, lg, ck
    torch.cuda.empty_cache()

    # ---- tree all-reduce of W row-parallel partials (simulated ranks, one GPU's HBM) -------
    E = M * 4096
    ar = {}
    for W in (2, 4, 8):
        parts = [torch.randn(E, device=dev, generator=g) for _ in range(W)]
        y = torch.empty(E, device=dev)
        grp = tb.DeviceGroup(W)
        ms = ev_ms(lambda: tb.tree_all_reduce(grp, parts), reps)
        ar[f"W{W}"] = line("allreduce_kernel (Algorithm 2 order)", 4.0 * (W + 1) * E, ms, peak, f"allreduce_W{W}")
        del parts, y
    out["tree_all_reduce_local"] = ar
    return out


if __name__ == "__main__":
    print(json.dumps(run()))
