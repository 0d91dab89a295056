"""oracle/gen_golden.py -- regenerate tests/golden/reference_golden.json.

TEST INFRASTRUCTURE.  Runs the UNMODIFIED reference library
(oracle/_ref/libtbik_ref.so, built from /root/reference/proj/src by
oracle/Makefile) on seeded inputs and records fingerprints / bit patterns.
The committed JSON pins both our C oracle (tests/test_oracle.py) and the GPU
kernels (tests/test_gpu_*.py) without needing /root/reference at run time.

Inputs are regenerated from the reference Rng (rng.hpp) by seed/stream, so
only fingerprints (bit_fingerprint, matrix.cpp:143-161) and a few raw values
are stored.  Usage:  python oracle/gen_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path[0] = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
from oracle.oracle import RefLib, OracleError  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "reference_golden.json")


def hexf(x) -> str:
    return "0x%08x" % int(np.float32(x).view(np.uint32))


def write_tbik_io_case(r: RefLib) -> None:
    """Golden I/O in the reference's own TBIK file format (matrix.cpp:211-233),
    written by the reference's matrix_write: a ragged-K tree_matmul case
    (K = 1000 -> 4 tiles of block_k 256, the last 232 wide) with its inputs and
    the reference output; diffable byte for byte against a GPU run."""
    d = os.path.join(os.path.dirname(OUT), "tbik_io")
    os.makedirs(d, exist_ok=True)
    a = r.random_normal(11, 1, 8, 1000, "bf16")
    b = r.random_normal(11, 2, 1000, 64, "bf16")
    c = r.tree_matmul(a, b, 256)
    for name, m in (("a", a), ("b", b), ("c_tree", c)):
        st = r.matrix_write(os.path.join(d, f"{name}.tbik"), m)
        if st:
            raise OracleError(f"ref_matrix_write failed: {st}")


def main() -> None:
    r = RefLib()
    g: dict = {"generator": "oracle/gen_golden.py over oracle/_ref/libtbik_ref.so "
                            "(unmodified /root/reference/proj/src)"}

    # RNG stream pins (rng.hpp:15-60, matrix.cpp:163-181).
    v = r.random_normal(1, 1, 1, 16, "f32")
    g["rng_f32_seed1_stream1_first16"] = [hexf(x) for x in v[0]]
    vb = r.random_normal(1, 2, 1, 16, "bf16")
    g["rng_bf16_seed1_stream2_first16"] = [int(x) for x in vb[0]]

    # Planner table (matmul.cpp:24-67).
    plans = []
    for K, bk, kf, cmax in [(14336, 256, 0, 8), (14336, 128, 0, 8), (25600, 256, 0, 8),
                            (25600, 128, 0, 8), (4096, 256, 0, 8), (6144, 256, 0, 8),
                            (8192, 256, 0, 8), (4096, 256, 0, 32), (5120, 256, 0, 1),
                            (5120, 256, 0, 8), (1000, 64, 0, 4), (4096, 256, 2, 8),
                            (4096, 256, 3, 1), (1, 1, 0, 1), (4096, 256, 0, 3)]:
        try:
            p = r.plan_blocks(K, bk, kf, cmax)
            plans.append({"K": K, "block_k": bk, "k_first": kf, "c_max": cmax, "status": 0,
                          "plan": list(p)})
        except OracleError as e:
            plans.append({"K": K, "block_k": bk, "k_first": kf, "c_max": cmax,
                          "status": e.code, "plan": None})
    g["plans"] = plans

    shards = []
    for K, bk, tp, cmax in [(14336, 256, 8, 8), (4096, 256, 4, 8), (1000, 64, 4, 4),
                            (14336, 256, 16, 8), (25600, 128, 8, 8)]:
        try:
            shards.append({"K": K, "block_k": bk, "tp": tp, "c_max": cmax, "status": 0,
                           "bounds": r.row_shard_plan(K, bk, 0, tp, cmax)})
        except OracleError as e:
            shards.append({"K": K, "block_k": bk, "tp": tp, "c_max": cmax, "status": e.code,
                           "bounds": None})
    g["row_shards"] = shards

    # Config 1 (BASELINE configs[0]): 64x4096x4096 bf16, TP 1/2/4/8.
    a = r.random_normal(1, 1, 64, 4096)
    b = r.random_normal(1, 2, 4096, 4096)
    g["config1"] = {
        "M": 64, "K": 4096, "N": 4096, "block_k": 256, "c_max": 8,
        "row_parallel_fingerprint": {str(tp): "0x%016x" % r.fingerprint(
            r.row_parallel_forward(a, b, tp)) for tp in (1, 2, 4, 8)},
        "global_tree_fingerprint": "0x%016x" % r.fingerprint(r.global_tree_matmul(a, b)),
    }

    # Llama down_proj (configs[1]) at M=1 and M=16, TP 1 and 8.
    a16 = r.random_normal(1, 1, 16, 14336)
    a1 = np.ascontiguousarray(r.random_normal(1, 1, 1, 14336))
    w = r.random_normal(1, 2, 14336, 4096)
    c1 = r.row_parallel_forward(a1, w, 1)
    c16 = r.row_parallel_forward(a16, w, 8)
    seq1 = r.baseline_row_parallel_forward(a1, w, 1)
    g["llama_down_proj"] = {
        "K": 14336, "N": 4096, "block_k": 256, "c_max": 8,
        "M1_fingerprint_tp1": "0x%016x" % r.fingerprint(c1),
        "M1_fingerprint_tp8": "0x%016x" % r.fingerprint(r.row_parallel_forward(a1, w, 8)),
        "M1_c00": hexf(c1[0, 0]),
        "M1_row0_first8": [hexf(x) for x in c1[0, :8]],
        "M16_fingerprint_tp8": "0x%016x" % r.fingerprint(c16),
        "M16_row0_equals_M1": bool(np.array_equal(c16[0].view(np.uint32), c1[0].view(np.uint32))),
        "M1_sequential_baseline_fingerprint": "0x%016x" % r.fingerprint(seq1),
        "M1_sequential_c00": hexf(seq1[0, 0]),
    }

    # Small ragged / f32 / k_first cases: full outputs are cheap to pin by fingerprint.
    small = []
    for (M, K, N, bk, kf, dt, seed) in [(5, 1000, 37, 64, 0, "bf16", 3), (3, 777, 19, 16, 0, "f32", 4),
                                        (7, 4096, 130, 256, 0, "bf16", 5), (2, 6144, 64, 256, 0, "bf16", 6),
                                        (4, 3000, 33, 100, 0, "f32", 7), (9, 512, 65, 32, 4, "bf16", 8)]:
        aa = r.random_normal(seed, 1, M, K, dt)
        bb = r.random_normal(seed, 2, K, N, dt)
        out = {"M": M, "K": K, "N": N, "block_k": bk, "k_first": kf, "dtype": dt, "seed": seed,
               "tree_matmul_fingerprint": "0x%016x" % r.fingerprint(r.tree_matmul(aa, bb, bk, kf)),
               "sequential_fingerprint": "0x%016x" % r.fingerprint(r.sequential_matmul(aa, bb))}
        rp = {}
        for tp in (1, 2, 4):
            try:
                rp[str(tp)] = "0x%016x" % r.fingerprint(r.row_parallel_forward(aa, bb, tp, bk, kf, 4))
            except OracleError as e:
                rp[str(tp)] = "error:%d" % e.code
        out["row_parallel_cmax4"] = rp
        small.append(out)
    g["small_cases"] = small

    # Tree all-reduce (collective.cpp:52-92) and ring stand-in (:94-106).
    ar = []
    for W in (1, 2, 4, 8):
        contrib = np.stack([r.random_normal(9, 1000 * W + k, 1, 257, "f32")[0] for k in range(W)])
        ar.append({"W": W, "elems": 257, "seed": 9,
                   "tree_fingerprint": "0x%016x" % r.fingerprint(r.tree_all_reduce(contrib)[None, :]),
                   "ring_fingerprint": "0x%016x" % r.fingerprint(r.ring_reduce(contrib)[None, :])})
    g["all_reduce"] = ar

    # Reference sequential rmsnorm (demo.cpp:11-34).
    x = r.random_normal(11, 1, 8, 4096)
    gamma = r.random_normal(11, 2, 1, 4096, "f32", 1.0, 0.02)[0]
    g["rmsnorm_seq"] = {"rows": 8, "cols": 4096, "seed": 11, "eps": 1e-5,
                        "fingerprint": "0x%016x" % r.fingerprint(r.rmsnorm(x, gamma, 1e-5))}

    # Witnesses (witness.cpp:10-71).
    na = r.nonassoc_witness()
    fw = r.fma_witness()
    seed, la, lb, lo = r.leaf_order_witness()
    g["witness"] = {"nonassoc": [hexf(v) for v in na], "fma": [hexf(v) for v in fw],
                    "leaf_order_seed": seed, "leaf_order": [hexf(v) for v in lo]}

    # Baseline kernel divergence (runner.cpp:216-237), f32 4x4096 . 4096x8 seed 1.
    a4 = r.random_normal(1, 1, 4, 4096, "f32")
    b8 = r.random_normal(1, 2, 4096, 8, "f32")
    g["baseline_divergence"] = {str(tp): "0x%016x" % r.fingerprint(
        r.baseline_row_parallel_forward(a4, b8, tp)) for tp in (1, 2, 4, 8)}

    ok, fails = r.check_theorem1_exhaustive(6, 100)
    g["theorem1_exhaustive"] = {"pass": ok, "failures": fails}
    ok, diffs = r.check_collective_symmetry(8, 8)
    g["collective_symmetry"] = {"pass": ok, "diffs": diffs}

    write_tbik_io_case(r)

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
        f.write("\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
