#!/usr/bin/env python
"""bench.py -- TBIK row-parallel GEMM (+ fixed-order tree all-reduce) on B200.

Workload (BASELINE.json configs[1]): the Llama-3.1-8B-shaped row-parallel
down_proj, K = 14336, N = 4096, M = 4096 tokens (16 x 256-token prompts),
bf16 inputs, f32 TBIK output, tensor-core leaves (TBIK_LEAF_TCGEN05,
block_k = 256, k_first = 7, 8 leaf groups).  With --gpus N the K dimension is
sharded with make_row_shard_plan (layers.cpp:23-46) over N processes, each
GPU runs the TBIK GEMM on its K range straight into its peer-visible buffer
and the partials meet in the NVLink tree all-reduce (strong scaling: the total
work is fixed).  A "step" is one row-parallel forward over the whole batch.

One JSON line (rank 0):
  value           whole-job TFLOP/s = 2*M*N*K / device time per step (max over ranks)
  e2e             same metric through the C ABI with HOST buffers: per step the
                  H2D copy of x (pinned) and the D2H read of y are inside the timed region
  roofline        the dominant kernel (tc_tree_gemm_kernel): algorithmic FLOPs per
                  launch / its CUDA-event duration vs MEASURED_PEAKS bf16 (burst)
  cpu_baseline    the unmodified reference library (oracle/_ref) on this host's cores
  noninvariant    cuBLAS bf16 GEMM (+ NCCL bf16 all-reduce at N > 1): the price of determinism
  sweep           M = 1 .. 4096 for the TC leaf, the exact (FMA) leaf and cuBLAS (rank 0, N = 1)
  tp_invariance   simulated TP = 1/2/4/8 bit-identity on this GPU (checked every run)
`--impl reference` times the reference's own CPU row_parallel_forward instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_FULL, N_OUT = 14336, 4096
METRIC = "TBIK row-parallel GEMM TFLOP/s at TP=1/2/4/8; bit-exact logits across TP"
WORKLOAD = "llama3.1-8b down_proj row-parallel (K=14336, N=4096) + tree all-reduce"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["tbik", "reference"], default="tbik")
    ap.add_argument("--m", type=int, default=4096)
    ap.add_argument("--leaf", choices=["tc", "fma"], default="tc")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-forward", action="store_true",
                    help="skip the full Llama-3.1-8B forward (logits bit-identity across TP)")
    ap.add_argument("--cpu-m", type=int, default=256,
                    help="rows of the bounded CPU sample (the reference's rate is ~3x lower at M=16)")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


class StdoutToStderr:
    """Route fd 1 to fd 2 while native libraries initialise (NCCL prints its version
    banner on stdout): the bench's stdout carries exactly one JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p["hbm_gbs"], "measured (MEASURED_PEAKS.json, burst bf16)"
    except Exception:  # noqa: BLE001
        return 1590.0, 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic_key(key):
    """dram bytes (read + write) per launch from the committed ncu capture
    (profiles/ncu_traffic.json, tools/traffic_capture.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:  # noqa: BLE001
        return None


def load_traffic(M, tp):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    return load_traffic_key(f"M{M}_tp{tp}")


class Clocks:
    """nvidia-smi sampler running DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
            out = ""
        sms, mx, reasons, samples = [], None, set(), 0
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            samples += 1
            try:
                sm = float(f[1])
                mx = float(f[2])
            except ValueError:
                continue
            sms.append(sm)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        sms.sort()
        busy = [s for s in sms if s > 500] or sms
        med = busy[len(busy) // 2] if busy else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": samples}


def ev_time_flushed(fn, reps):
    """Device time (ms) per call of fn, each call preceded by an L2 eviction that
    READS 256 MB (no dirty lines left to write back inside the timed call)."""
    import torch
    flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    sink = torch.empty((), device="cuda")
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
    del flush
    return tot / reps


def ev_time(fn, reps, stream=None):
    """Device time (ms) per call of fn with CUDA events on the current stream."""
    import torch
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


# ------------------------------------------------------------------------------------
# reference arm: the unmodified reference library on the host cores
# ------------------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_sample(tp: int, m_sample: int, budget_s: float, min_reps: int = 1):
    import numpy as np

    from oracle.oracle import RefLib
    ref = RefLib()
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    a = ref.random_normal(1, 1, m_sample, K_FULL)
    w = ref.random_normal(1, 2, K_FULL, N_OUT)
    times = []
    t_start = time.perf_counter()
    while len(times) < min_reps or (time.perf_counter() - t_start < budget_s and len(times) < 50):
        t0 = time.perf_counter()
        y = ref.row_parallel_forward(a, w, tp)
        times.append(time.perf_counter() - t0)
    best = min(times)
    flops = 2.0 * m_sample * N_OUT * K_FULL
    fp = ref.fingerprint(np.ascontiguousarray(y))
    # one-thread point: a single call on M=1 row
    ref.set_threads(1)
    a1 = a[:1].copy()
    t0 = time.perf_counter()
    ref.row_parallel_forward(a1, w, tp)
    t1 = time.perf_counter() - t0
    ref.set_threads(threads)
    return {"value": flops / best / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(), "one_thread_m1_tflops": 2.0 * N_OUT * K_FULL / t1 / 1e12,
            "sample": f"row_parallel_forward(DeviceGroup({tp})) on M={m_sample} rows of the "
                      f"{K_FULL}x{N_OUT} down_proj, bf16 N(0,1) Rng(1,1)/(1,2), best of {len(times)} "
                      f"wall-clock runs ({sum(times):.1f} s of CPU work), TBIK_THREADS={threads}",
            "fingerprint": "0x%016x" % fp, "seconds_per_call": best}


def run_reference(args):
    rank, _, world = env_rank()
    if rank != 0:
        return
    tp = args.gpus
    m_sample = args.cpu_m
    import numpy as np

    from oracle.oracle import RefLib
    ref = RefLib()
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    a = ref.random_normal(1, 1, m_sample, K_FULL)
    w = ref.random_normal(1, 2, K_FULL, N_OUT)
    for _ in range(args.warmup):
        ref.row_parallel_forward(a, w, tp)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        y = ref.row_parallel_forward(a, w, tp)
    dt = (time.perf_counter() - t0) / args.steps
    flops = 2.0 * m_sample * N_OUT * K_FULL
    value = flops / dt / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (reference Rng, N(0,1) bf16)",
        "config": {"workload": WORKLOAD, "M": m_sample, "M_note": "bounded CPU sample of the M=4096 workload",
                   "K": K_FULL, "N": N_OUT, "tp": tp, "parallelism": f"tp{tp} (simulated ranks on host threads)",
                   "block_k": 256},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"row_parallel_forward(DeviceGroup({tp})) M={m_sample} rows per step"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "fingerprint": "0x%016x" % ref.fingerprint(np.ascontiguousarray(y)),
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------------------
# TBIK arm
# ------------------------------------------------------------------------------------
def sharded_forward(group, rank, world, barrier, max_over_ranks, batch=4, seq=256, reps=3):
    """Llama-3.1-8B (32 layers, random init) prefill of batch x seq tokens with W real
    ranks (model.ShardedDecoder: each process holds its shards; row-parallel tree
    all-reduce, all-gather and (m, s) merge over the PeerGroup), timed as the max
    over ranks; rank 0 checks the all-gathered logits / log-probs against the
    single-GPU TP = 1 forward of the full weights."""
    import torch

    from paper_2511_17826_b200 import model as mdl
    cfg = mdl.llama31_8b()
    dec = mdl.ShardedDecoder(cfg, group, seed=3)
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    tokens = torch.randint(0, cfg.vocab, (batch, seq), device="cuda", generator=g)
    M = batch * seq

    def step():
        logits = dec.forward(tokens)
        return logits, dec.log_probs(logits, full=True)

    step()
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev_time(step, reps))
    logits_r, (_, lp_r, _) = step()
    logits = dec.gather(logits_r)
    lp = dec.gather(lp_r)
    torch.cuda.synchronize()
    out = {"model": cfg.name, "layers": cfg.n_layers, "batch": batch, "seq": seq, "tokens": M, "tp": world,
           "ms": ms, "tokens_per_s": M / (ms * 1e-3),
           "path": "ShardedDecoder: one process per GPU, rank-local weight shards, PeerGroup collectives"}
    del dec
    torch.cuda.empty_cache()
    if rank == 0:
        full = mdl.TbikDecoder(cfg, mdl.random_weights(cfg, seed=3))
        ref_logits = full.forward(tokens, 1)
        _, ref_lp, _ = full.log_probs(ref_logits, 1, full=True)
        torch.cuda.synchronize()
        out["logits_bit_identical_to_tp1"] = bool(torch.equal(logits.view(torch.int32), ref_logits.view(torch.int32)))
        out["logprobs_bit_identical_to_tp1"] = bool(torch.equal(lp.view(torch.int32), ref_lp.view(torch.int32)))
        del full, ref_logits, ref_lp
        torch.cuda.empty_cache()
    barrier()
    return out


def run_tbik(args):
    import torch
    import torch.distributed as dist

    import paper_2511_17826_b200 as tb

    rank, local_rank, world = env_rank()
    if world != args.gpus:
        world = args.gpus if world == 1 else world
    # TBIK_BENCH_SHARE_GPU=1: every rank on device 0 with a gloo control plane -- a
    # functional check of the N > 1 path on a one-GPU box (timings meaningless).
    share = os.environ.get("TBIK_BENCH_SHARE_GPU") == "1"
    dev_index = 0 if share else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        with StdoutToStderr():
            if share:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=dev)
    leaf = tb.LEAF_TCGEN05 if args.leaf == "tc" else tb.LEAF_FMA
    cfg = tb.BlockConfig(64, 256, 128, 0)
    M = args.m
    shard = tb.make_row_shard_plan(K_FULL, cfg, world, 8)
    kb, ke = shard.bounds[rank]
    Kr = ke - kb
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    w_full_rows = torch.randn(K_FULL, N_OUT, device=dev, generator=g, dtype=torch.float32)
    w = w_full_rows[kb:ke].to(torch.bfloat16).contiguous()
    del w_full_rows
    x_full = torch.randn(M, K_FULL, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
    x = x_full[:, kb:ke].contiguous()
    y = torch.empty(M, N_OUT, device=dev, dtype=torch.float32)

    group = None
    if world > 1:
        group = tb.PeerGroup(world, rank, dev_index, M * N_OUT, dist)

        def step():
            group.row_parallel_forward(x, w, K_FULL, cfg, 8, leaf, out=y)
    else:
        def step():
            tb.tree_matmul(x, w, cfg, leaf, out=y)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warmup + timed region -----------------------------------------------------
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(dev_index)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    launches0 = tb.launch_count()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(args.steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    launches = tb.launch_count() - launches0
    y_step = y.clone()  # the step's result (y is reused below by the single-GPU roofline timing)
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    flops = 2.0 * M * N_OUT * K_FULL
    value = flops / (ms * 1e-3) / 1e12

    # ---- the dominant kernel on its own (roofline) -----------------------------------
    k_ms = ev_time(lambda: tb.tree_matmul(x, w, cfg, leaf, out=y), max(args.steps, 5))
    k_name = tb.last_kernel() or ("tc_tree_gemm_kernel" if leaf else "fma_tree_gemm_kernel")
    k_flops = 2.0 * M * N_OUT * Kr
    achieved = k_flops / (k_ms * 1e-3) / 1e12
    peak_tf, peak_hbm, peak_src = load_peaks()
    bytes_alg = 2.0 * M * Kr + 2.0 * Kr * N_OUT + 4.0 * M * N_OUT
    intensity = k_flops / bytes_alg
    tensor_bound = intensity > peak_tf * 1e12 / (peak_hbm * 1e9)
    if tensor_bound:
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved / peak_tf}
    else:
        gbs = bytes_alg / (k_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": gbs, "peak": peak_hbm, "unit": "GB/s", "frac": gbs / peak_hbm}
    roof.update({"traffic": load_traffic(M, world), "kernel": k_name,
                 "kernel_ms": k_ms, "flops_per_launch": k_flops, "alg_bytes_per_launch": bytes_alg,
                 "peak_source": peak_src, "share_of_step": k_ms / ms if ms else None})

    # ---- e2e through the C ABI with host buffers ----------------------------------------
    # tbik_tree_matmul_hostio / tbik_group_row_parallel_forward_hostio: pinned host x in,
    # pinned host y out; the H2D of row chunk i+1, the GEMM (+ tree all-reduce) of chunk i
    # and the D2H of chunk i-1 overlap (bit-identical to the device call: batch invariance).
    x_host = x.cpu().pin_memory()
    y_host = torch.empty(M, N_OUT, dtype=torch.float32).pin_memory()

    def e2e_step():
        if group is not None:
            group.row_parallel_forward_hostio(x_host, w, K_FULL, cfg, 8, leaf, out=y_host)
        else:
            tb.tree_matmul_hostio(x_host, w, cfg, leaf, out=y_host)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e2e_same = bool(torch.equal(y_host.view(torch.int32), y_step.cpu().view(torch.int32)))
    barrier()
    e2e_ms = max_over_ranks(ev_time(e2e_step, max(args.steps // 2, 3)))
    e2e = {"value": flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
           "h2d_bytes_per_step": x_host.numel() * x_host.element_size(),
           "d2h_bytes_per_step": y_host.numel() * y_host.element_size(),
           "ms_per_step": e2e_ms, "bit_identical_to_device_call": e2e_same,
           "path": "pinned host x -> tbik_tree_matmul_hostio / tbik_group_row_parallel_forward_hostio (C ABI: "
                   "row-chunked H2D | GEMM + tree all-reduce | D2H on three streams) -> pinned host y"}

    # ---- non-invariant status quo: cuBLAS (+ NCCL all-reduce) ------------------------------------
    # tbik_baseline_cublas_nccl (C ABI): cuBLAS GEMM of this rank's shard, then NCCL's sum
    # all-reduce -- bf16 output + bf16 all-reduce (what a serving stack runs) and f32 output
    # + f32 all-reduce (the same bytes per rank as the TBIK tree all-reduce).  At N = 1 the
    # communicator has one rank (no transfer).
    import ctypes as C
    uid = (C.c_char * 128)()
    if rank == 0:
        tb.api.check(tb.lib.tbik_nccl_unique_id(uid))
    if world > 1:
        holder = [bytes(uid)]
        dist.broadcast_object_list(holder, src=0)
        uid = (C.c_char * 128).from_buffer_copy(holder[0])
    comm = C.c_void_p()
    if not share:
        with StdoutToStderr():
            tb.api.check(tb.lib.tbik_nccl_comm_create(world, rank, dev_index, uid, C.byref(comm)))
    yb = torch.empty(M, N_OUT, device=dev, dtype=torch.bfloat16)
    yf = torch.empty(M, N_OUT, device=dev, dtype=torch.float32)

    def cublas_step(out_f32):
        def f():
            if share:
                torch.matmul(x, w, out=yb)
                return
            o = yf if out_f32 else yb
            tb.api.check(tb.lib.tbik_baseline_cublas_nccl(comm, C.c_void_p(x.data_ptr()), 1, Kr,
                                                          C.c_void_p(w.data_ptr()), 1, N_OUT, C.c_void_p(o.data_ptr()),
                                                          M, N_OUT, Kr, 1 if out_f32 else 0,
                                                          C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return f

    noninv = {"path": "tbik_baseline_cublas_nccl: cuBLAS GEMM of the rank's K shard + NCCL sum all-reduce "
                      "(order not controlled: non-invariant)"}
    for key, out_f32 in (("bf16", False), ("f32", True)):
        fn = cublas_step(out_f32)
        for _ in range(3):
            fn()
        barrier()
        bms = max_over_ranks(ev_time(fn, max(args.steps, 5)))
        btf = flops / (bms * 1e-3) / 1e12
        noninv[key] = {"value": btf, "unit": "TFLOP/s", "ms_per_step": bms, "tbik_over_baseline": value / btf,
                       "out": f"{key} GEMM output + {key} all-reduce" if world > 1 else f"{key} GEMM output"}
    noninv["tbik_over_baseline"] = noninv["bf16"]["tbik_over_baseline"]
    if not share:
        tb.lib.tbik_nccl_comm_destroy(comm)
    del yf

    # ---- the tree all-reduce alone over NVLink (N > 1): algorithmic and bus bandwidth ---------
    collective_bw = None
    if group is not None:
        part = torch.randn(M * N_OUT, device=dev, generator=g)
        red = torch.empty_like(part)
        barrier()
        ar_ms = max_over_ranks(ev_time(lambda: group.tree_all_reduce(part, out=red), max(args.steps, 5)))
        alg = 4.0 * M * N_OUT / (ar_ms * 1e-3) / 1e9
        collective_bw = {"kernel": "tree all-reduce over peer memory (one-shot < 1 MiB, else reduce-scatter + push)",
                         "bytes_per_rank": 4 * M * N_OUT, "ms": ar_ms, "alg_GBps": alg,
                         "bus_GBps": alg * 2 * (world - 1) / world, "nvlink_peak_GBps_per_direction": 900.0,
                         "bus_frac": alg * 2 * (world - 1) / world / 900.0}
        del part, red

    # ---- TP invariance at the bench config (simulated ranks on this GPU), every run -----------
    # M = 4096 rows, the full down_proj: TP = 1/2/4/8 must give one bit pattern.
    tp_ok = None
    if rank == 0:
        wf = (torch.randn(K_FULL, N_OUT, device=dev, generator=g).to(torch.bfloat16) if world > 1
              else w)
        outs = [tb.row_parallel_forward(x_full, wf, tb.DeviceGroup(t), cfg, 8, leaf) for t in (1, 2, 4, 8)]
        tp_ok = {"M": M, "tp": [1, 2, 4, 8],
                 "bit_identical": all(torch.equal(outs[0].view(torch.int32), o.view(torch.int32)) for o in outs[1:])}
        del wf, outs

    # ---- M sweep (rank 0, N = 1) ----------------------------------------------------------------
    sweep = None
    if rank == 0 and world == 1 and not args.no_sweep:
        sweep = {"M": [], "tbik_tc_tflops": [], "tbik_fma_tflops": [], "cublas_bf16_tflops": [],
                 "timing": "per call, after a 256 MB read that evicts W (117 MB) from L2"}
        for m in (1, 16, 64, 256, 1024, 4096):
            xm = x[:m].contiguous()
            ym = torch.empty(m, N_OUT, device=dev)
            yc = torch.empty(m, N_OUT, device=dev, dtype=torch.bfloat16)
            f = 2.0 * m * N_OUT * K_FULL
            reps = 20 if m <= 1024 else 10
            t_tc = ev_time_flushed(lambda: tb.tree_matmul(xm, w, cfg, tb.LEAF_TCGEN05, out=ym), reps)
            if m <= 1024:
                t_fma = ev_time_flushed(lambda: tb.tree_matmul(xm, w, cfg, tb.LEAF_FMA, out=ym), max(reps // 4, 2))
            else:
                t_fma = None
            t_cb = ev_time_flushed(lambda: torch.matmul(xm, w, out=yc), reps)
            sweep["M"].append(m)
            sweep["tbik_tc_tflops"].append(f / (t_tc * 1e-3) / 1e12)
            sweep["tbik_fma_tflops"].append(f / (t_fma * 1e-3) / 1e12 if t_fma else None)
            sweep["cublas_bf16_tflops"].append(f / (t_cb * 1e-3) / 1e12)

    # ---- per-rank GEMM of each TP shard (rank 0, N = 1): the compute side of TP = 2/4/8 ----
    tp_shards = None
    if rank == 0 and world == 1 and not args.no_sweep:
        tp_shards = {"note": "rank 0's row-parallel shard GEMM (K/tp, global k_first) on this GPU; the NVLink "
                             "all-reduce is not in these numbers (one GPU)", "tp": [], "per_rank_tflops": [],
                     "per_rank_ms": []}
        for t in (1, 2, 4, 8):
            sp = tb.make_row_shard_plan(K_FULL, cfg, t, 8)
            kb0, ke0 = sp.bounds[0]
            xs_t = x_full[:, kb0:ke0].contiguous()
            ws_t = w[kb0:ke0].contiguous() if world == 1 else None
            cfg_t = tb.BlockConfig(64, 256, 128, tb.plan_blocks(K_FULL, cfg, 8).k_first)
            yt = torch.empty(M, N_OUT, device=dev)
            ms_t = ev_time(lambda: tb.tree_matmul(xs_t, ws_t, cfg_t, leaf, out=yt), max(args.steps, 5))
            tp_shards["tp"].append(t)
            tp_shards["per_rank_ms"].append(ms_t)
            tp_shards["per_rank_tflops"].append(2.0 * M * N_OUT * (ke0 - kb0) / (ms_t * 1e-3) / 1e12)
            tp_shards.setdefault("traffic", []).append(load_traffic(M, 1) if t == 1 else
                                                        load_traffic_key(f"M{M}_shard_tp{t}"))
            del xs_t, ws_t, yt

    # ---- the metric's second half: bit-exact logits across TP on the Llama forward ----
    forward = None
    if rank == 0 and world == 1 and not args.no_forward:
        del w, x, x_full, y, yb, x_host, y_host, y_step
        torch.cuda.empty_cache()
        from tools.forward_bench import run as forward_run
        try:
            forward = forward_run("llama3.1-8b", 32, 4, 256, reps=3, tps=(1, 2, 4, 8))
        except Exception as e:  # noqa: BLE001 -- the headline line must still print
            forward = {"error": f"{type(e).__name__}: {e}"[:300]}
            torch.cuda.synchronize()

    # ---- the north-star forward at real TP (N > 1): one process per GPU, rank shards only ----
    forward_tp = None
    if world > 1 and not args.no_forward:
        del w, x, x_full, y, yb, x_host, y_host, y_step
        torch.cuda.empty_cache()
        try:
            forward_tp = sharded_forward(group, rank, world, barrier, max_over_ranks)
        except Exception as e:  # noqa: BLE001 -- the headline line must still print
            forward_tp = {"error": f"{type(e).__name__}: {e}"[:300]}

    rowops = None
    if rank == 0 and world == 1 and not args.no_forward:
        torch.cuda.empty_cache()
        from tools.rowops_bench import run as rowops_run
        try:
            rowops = rowops_run(reps=10, tps=(1, 8))
        except Exception as e:  # noqa: BLE001
            rowops = {"error": f"{type(e).__name__}: {e}"[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference_sample(1, args.cpu_m, budget_s=12.0, min_reps=2)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: device-generated N(0,1) weights/activations rounded to bf16 (random init, "
                    "Llama-3.1-8B down_proj shape)",
            "config": {"workload": WORKLOAD, "M": M, "K": K_FULL, "N": N_OUT, "tp": world,
                       "parallelism": f"tp{world} row-parallel", "leaf": args.leaf, "block_k": cfg.block_k,
                       "k_first": tb.plan_blocks(K_FULL, cfg, 8).k_first, "c_max": 8,
                       "l2": "no flush: per-step inputs+output (x 117 MB + W 117 MB + y 67 MB at tp1) exceed the 126 MB L2"},
            "roofline": roof, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "noninvariant": noninv, "tp_invariance_bit_identical": tp_ok, "sweep": sweep,
            "tp_shard_gemm": tp_shards,
            "collective": None if group is None else {
                "path": "fused: one tcgen05 kernel = GEMM + tile-flag tree all-reduce over peer memory"
                        if group.fused_count() > 0 else "GEMM, then tree all-reduce kernels",
                "fused_calls": group.fused_count(), "tree_all_reduce_alone": collective_bw},
            "forward_tp": forward_tp,
            "cpu_baseline": cpu,
            "forward": forward,
            "rowops_c5": rowops,
        }
        print(json.dumps(line))
    if group is not None:
        barrier()
        group.close()
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without a torchrun environment: launch the N
    ranks ourselves exactly as the driver does (torch.distributed.run, one process
    per GPU, rendezvous on 127.0.0.1) and pass rank 0's JSON line through."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)  # rank 0 alone works; needs no process group
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_tbik(args)


if __name__ == "__main__":
    main()
