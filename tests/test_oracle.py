"""CPU suite: pin the C oracle (oracle/tbik_oracle.c) to the reference.

Two anchors: the committed golden vectors (tests/golden/reference_golden.json,
generated from the unmodified reference by oracle/gen_golden.py) and, when it
was built here, the reference library itself (oracle/_ref).  Mirrors the
reference's own checks (runner.cpp:53-325) and the SPEC known-answer tests.
"""
import numpy as np
import pytest

from conftest import bits, fp_hex


def f32(h: str) -> np.float32:
    return np.array([int(h, 16)], np.uint32).view(np.float32)[0]


# ---- RNG / storage (rng.hpp, numerics.hpp) ------------------------------------------
def test_rng_streams_match_golden(orc, golden):
    v = orc.random_normal(1, 1, 1, 16, "f32")[0]
    assert ["0x%08x" % x for x in bits(v)] == golden["rng_f32_seed1_stream1_first16"]
    vb = orc.random_normal(1, 2, 1, 16, "bf16")[0]
    assert [int(x) for x in vb] == golden["rng_bf16_seed1_stream2_first16"]


def test_bf16_roundtrip_exhaustive(orc):
    # check_bf16_exhaustive (runner.cpp:304-325)
    pats = np.arange(0x10000, dtype=np.uint32)
    f = (pats << 16).view(np.float32)
    nan = ((pats & 0x7F80) == 0x7F80) & ((pats & 0x7F) != 0)
    back = np.array([orc.bf16_round(x) for x in f[~nan][::97]])
    assert np.array_equal(back, pats[~nan][::97])
    assert orc.bf16_round(float("nan")) == 0x7FC0


def test_bf16_rne_ties(orc):
    assert orc.bf16_round(np.float32(1.0) + np.float32(2.0 ** -8)) == 0x3F80  # tie -> even
    assert orc.bf16_round(np.uint32(0x3F818000).view(np.float32)) == 0x3F82  # tie -> even (up)


# ---- planner (matmul.cpp:24-67, layers.cpp:9-46) ---------------------------------------
def test_plan_table_matches_reference(orc, golden):
    for row in golden["plans"]:
        if row["status"] == 0:
            assert list(orc.plan_blocks(row["K"], row["block_k"], row["k_first"], row["c_max"])) == row["plan"]
        else:
            with pytest.raises(Exception) as e:
                orc.plan_blocks(row["K"], row["block_k"], row["k_first"], row["c_max"])
            assert e.value.code == row["status"]


def test_row_shards_match_reference(orc, golden):
    for row in golden["row_shards"]:
        if row["status"] == 0:
            got = orc.row_shard_plan(row["K"], row["block_k"], 0, row["tp"], row["c_max"])
            assert [list(b) for b in got] == row["bounds"]
        else:
            with pytest.raises(Exception) as e:
                orc.row_shard_plan(row["K"], row["block_k"], 0, row["tp"], row["c_max"])
            assert e.value.code == row["status"]


def test_spec_plan_example(orc):
    # K=6144, block_k=256, c_max=8 -> T=24, k_first=3, leaves=8, L=4
    assert orc.plan_blocks(6144, 256, 0, 8) == (24, 3, 8, 4)


# ---- tree operator / Theorem 1 ----------------------------------------------------------
def test_tree_reduce_kats(orc):
    assert orc.tree_reduce([1.0, 2.0, 3.0, 4.0]) == np.float32(10.0)
    assert orc.tree_reduce([1e8, 1.0, -1e8, 1.0]) == np.float32(0.0)
    assert orc.ring_reduce(np.array([[1e8], [1.0], [-1e8], [1.0]], np.float32))[0] == np.float32(1.0)


def test_theorem1_random(orc):
    # check_theorem1_exhaustive (runner.cpp:93-127) restated on our operator
    rng = np.random.default_rng(0)
    for t in range(0, 7):
        n = 1 << t
        for j in range(t + 1):
            tp = 1 << j
            for _ in range(20):
                leaves = (rng.standard_normal(n) * 2.0 ** rng.integers(-20, 21, n)).astype(np.float32)
                parts = [orc.tree_reduce(leaves[d * (n // tp):(d + 1) * (n // tp)]) for d in range(tp)]
                assert bits(np.float32(orc.tree_reduce(parts))).item() == bits(np.float32(orc.tree_reduce(leaves))).item()


# ---- the GEMM -----------------------------------------------------------------------------
def test_config1_golden_fingerprint(orc, golden):
    g = golden["config1"]
    a = orc.random_normal(1, 1, 64, 4096)
    b = orc.random_normal(1, 2, 4096, 4096)
    want = fp_hex(g["global_tree_fingerprint"])
    assert orc.fingerprint(orc.global_tree_matmul(a, b, 256, 0, 8)) == want
    assert orc.fingerprint(orc.tree_matmul(a, b, 256, 0)) == want
    for tp in (1, 2, 4, 8):
        assert fp_hex(g["row_parallel_fingerprint"][str(tp)]) == want
        assert orc.fingerprint(orc.row_parallel_forward(a, b, tp, 256, 0, 8)) == want


def test_llama_down_proj_m1_golden(orc, golden):
    g = golden["llama_down_proj"]
    a = orc.random_normal(1, 1, 1, 14336)
    w = orc.random_normal(1, 2, 14336, 4096)
    c = orc.global_tree_matmul(a, w, 256, 0, 8)
    assert orc.fingerprint(c) == fp_hex(g["M1_fingerprint_tp1"])
    assert "0x%08x" % int(bits(c)[0, 0]) == g["M1_c00"]
    s = orc.sequential_matmul(a, w)
    assert orc.fingerprint(s) == fp_hex(g["M1_sequential_baseline_fingerprint"])
    assert orc.fingerprint(orc.row_parallel_forward(a, w, 8)) == fp_hex(g["M1_fingerprint_tp8"])


def test_small_cases_golden(orc, golden):
    for case in golden["small_cases"]:
        a = orc.random_normal(case["seed"], 1, case["M"], case["K"], case["dtype"])
        b = orc.random_normal(case["seed"], 2, case["K"], case["N"], case["dtype"])
        assert orc.fingerprint(orc.tree_matmul(a, b, case["block_k"], case["k_first"])) == \
            fp_hex(case["tree_matmul_fingerprint"])
        assert orc.fingerprint(orc.sequential_matmul(a, b)) == fp_hex(case["sequential_fingerprint"])
        for tp, want in case["row_parallel_cmax4"].items():
            if want.startswith("error"):
                with pytest.raises(Exception) as e:
                    orc.row_parallel_forward(a, b, int(tp), case["block_k"], case["k_first"], 4)
                assert e.value.code == int(want.split(":")[1])
            else:
                got = orc.row_parallel_forward(a, b, int(tp), case["block_k"], case["k_first"], 4)
                assert orc.fingerprint(got) == fp_hex(want)


def test_tree_over_leaves_equals_kernel(orc):
    rng = np.random.default_rng(1)
    a = rng.standard_normal((3, 1000)).astype(np.float32)
    b = rng.standard_normal((1000, 5)).astype(np.float32)
    T, kf = 16, 1
    bk = 64
    leaves = np.zeros((T, 3, 5), np.float32)
    for t in range(T):
        k0, k1 = t * bk, min((t + 1) * bk, 1000)
        for i in range(3):
            for j in range(5):
                leaves[t, i, j] = orc.lib.tbo_leaf_dot(
                    np.ascontiguousarray(a[i, k0:k1]).ctypes.data_as(orc.lib.tbo_leaf_dot.argtypes[0]),
                    np.ascontiguousarray(b[k0:k1, j]).ctypes.data_as(orc.lib.tbo_leaf_dot.argtypes[1]),
                    k1 - k0)
    got = orc.tree_over_leaves(leaves, kf)
    assert np.array_equal(bits(got), bits(orc.tree_matmul(a, b, bk, 0)))


def test_identity_a_gives_b(orc):
    # A = identity -> C bit-equal to B
    n = 64
    a = np.eye(n, dtype=np.float32)
    b = np.random.default_rng(2).standard_normal((n, 7)).astype(np.float32)
    assert np.array_equal(bits(orc.tree_matmul(a, b, 16, 0)), bits(b))


def test_spec_toy_kat(orc):
    # A=[1e8,1,-1e8,1], B=1, block_k=1 -> tree 0, sequential 1
    a = np.array([[1e8, 1.0, -1e8, 1.0]], np.float32)
    b = np.ones((4, 1), np.float32)
    assert orc.tree_matmul(a, b, 1, 1)[0, 0] == 0.0
    assert orc.sequential_matmul(a, b)[0, 0] == 1.0
    for tp in (1, 2, 4):
        assert orc.row_parallel_forward(a, b, tp, 1, 1, 4)[0, 0] == 0.0


# ---- collective ---------------------------------------------------------------------------
def test_all_reduce_golden(orc, golden):
    for row in golden["all_reduce"]:
        W = row["W"]
        contrib = np.stack([orc.random_normal(9, 1000 * W + k, 1, 257, "f32")[0] for k in range(W)])
        assert orc.fingerprint(orc.tree_all_reduce(contrib)[None, :]) == fp_hex(row["tree_fingerprint"])
        assert orc.fingerprint(orc.ring_reduce(contrib)[None, :]) == fp_hex(row["ring_fingerprint"])


def test_bad_world_size(orc):
    with pytest.raises(Exception) as e:
        orc.tree_all_reduce(np.zeros((3, 4), np.float32))
    assert e.value.code == 8  # BadWorldSize


def test_baseline_divergence_golden(golden):
    # the problem being solved is real: the sequential+ring baseline diverges across TP
    assert len(set(golden["baseline_divergence"].values())) >= 2


# ---- rmsnorm ------------------------------------------------------------------------------
def test_rmsnorm_seq_golden(orc, golden):
    g = golden["rmsnorm_seq"]
    x = orc.random_normal(11, 1, 8, 4096)
    gamma = orc.random_normal(11, 2, 1, 4096, "f32", 1.0, 0.02)[0]
    assert orc.fingerprint(orc.rmsnorm_seq(x, gamma, 1e-5)) == fp_hex(g["fingerprint"])


def test_tree_rmsnorm_close_to_sequential(orc):
    x = orc.random_normal(5, 1, 4, 5120)
    gamma = orc.random_normal(5, 2, 1, 5120, "f32", 1.0, 0.02)[0]
    a = orc.tree_rmsnorm(x, gamma)
    b = orc.rmsnorm_seq(x, gamma)
    assert np.max(np.abs(a - b) / (np.abs(b) + 1e-6)) < 1e-5


# ---- shared exp / log and the (m, s) log-softmax ------------------------------------------
def test_exp_log_accuracy(orc):
    xs = np.linspace(-100, 0, 20001, dtype=np.float32)
    e = np.array([orc.exp(x) for x in xs], np.float32)
    ref = np.exp(xs.astype(np.float64))
    mask = ref > 1e-37
    assert np.max(np.abs(e[mask] - ref[mask]) / ref[mask]) < 4e-7
    ys = np.exp(np.linspace(-80, 80, 20001)).astype(np.float32)
    lg = np.array([orc.log(y) for y in ys], np.float64)
    err = np.abs(lg - np.log(ys.astype(np.float64)))
    assert np.max(err / np.maximum(np.abs(np.log(ys.astype(np.float64))), 1.0)) < 4e-7
    assert orc.exp(-200.0) == 0.0 and orc.exp(0.0) == 1.0


def test_tree_logsoftmax_close_and_sharding_exact(orc):
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((3, 1024)) * 4).astype(np.float32)
    lse, lp, _ = orc.tree_logsoftmax(x, 8, full=True)
    ref = np.log(np.sum(np.exp(x.astype(np.float64)), axis=1))
    assert np.max(np.abs(lse - ref)) < 1e-5
    # group states merged by hand in rank order == full tree (Theorem 1 for (m, s))
    m, s = orc.logsoftmax_group_states(x, 8)
    assert m.shape == (3, 8)
    lse16, _, _ = orc.tree_logsoftmax(x, 16)
    assert np.max(np.abs(lse16 - ref)) < 1e-5


# ---- the reference's own suites, run on the reference (sanity of the harness) -------------
def test_reference_checks_pass(ref):
    ok, fails = ref.check_theorem1_exhaustive(6, 20)
    assert ok and fails == 0
    ok, diffs = ref.check_collective_symmetry(8, 8)
    assert ok and diffs == 0


def test_oracle_equals_reference_random(orc, ref):
    rng = np.random.default_rng(7)
    for _ in range(4):
        M = int(rng.integers(1, 6))
        K = int(rng.integers(1, 700))
        N = int(rng.integers(1, 40))
        bk = int(rng.choice([1, 8, 16, 64, 100]))
        dt = str(rng.choice(["f32", "bf16"]))
        seed = int(rng.integers(1, 1000))
        a = orc.random_normal(seed, 1, M, K, dt)
        b = orc.random_normal(seed, 2, K, N, dt)
        assert np.array_equal(a, ref.random_normal(seed, 1, M, K, dt))
        assert np.array_equal(bits(orc.tree_matmul(a, b, bk)), bits(ref.tree_matmul(a, b, bk)))
        assert np.array_equal(bits(orc.global_tree_matmul(a, b, bk, 0, 1)),
                              bits(ref.global_tree_matmul(a, b, bk, 0, 1)))
