"""oracle/oracle.py -- ctypes loaders for the CPU checkers.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  Never imported by the
product package (paper_2511_17826_b200), which fails loudly without its CUDA
library instead of falling back here.

Two libraries:
  * ``Oracle``  -- oracle/libtbik_oracle.so, our plain-C restatement
                   (tbik_oracle.c, every function cites the reference file:line);
  * ``RefLib``  -- oracle/_ref/libtbik_ref.so, the unmodified reference library
                   compiled from /root/reference/proj/src plus ref_shim.cpp.
Both take/return numpy arrays.  dtype codes follow tbik::Dtype
(matrix.hpp:20): 0 = f32, 1 = bf16 (stored as uint16 bit patterns).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libtbik_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtbik_ref.so")

i64 = C.c_int64
u64 = C.c_uint64
f32 = C.c_float
vp = C.c_void_p
PF = C.POINTER(C.c_float)
PI64 = C.POINTER(C.c_int64)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: status {code}")
        self.code = code


def build() -> None:
    """Compile the checkers (idempotent; make decides what is stale)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 0
    if a.dtype == np.uint16:
        return 1
    raise TypeError(f"oracle matrices are float32 or uint16(bf16 bits), got {a.dtype}")


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(vp)


def _check(code: int, what: str) -> None:
    if code != 0:
        raise OracleError(code, what)


class _Lib:
    so_path = ""

    def __init__(self):
        if not os.path.exists(self.so_path):
            build()
        self.lib = C.CDLL(self.so_path)


class Oracle(_Lib):
    """Our C restatement (tbik_oracle.c)."""

    so_path = ORACLE_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.tbo_bf16_round.restype = C.c_uint16
        L.tbo_bf16_round.argtypes = [f32]
        L.tbo_random_normal.argtypes = [u64, u64, i64, i64, C.c_int, f32, f32, vp]
        L.tbo_fingerprint.restype = u64
        L.tbo_fingerprint.argtypes = [vp, C.c_int, i64, i64]
        L.tbo_plan_blocks.argtypes = [i64, i64, i64, i64, PI64]
        L.tbo_make_row_shard_plan.argtypes = [i64, i64, i64, C.c_int, i64, PI64]
        L.tbo_make_column_shard_plan.argtypes = [i64, C.c_int, PI64]
        L.tbo_tree_reduce.argtypes = [PF, i64, PF]
        L.tbo_leaf_dot.restype = f32
        L.tbo_leaf_dot.argtypes = [PF, PF, i64]
        L.tbo_tree_matmul.argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64, i64, i64, PF]
        L.tbo_global_tree_matmul.argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64, i64, i64, i64, PF]
        L.tbo_tree_over_leaves.argtypes = [PF, i64, i64, i64, PF]
        L.tbo_sequential_matmul.argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64, PF]
        L.tbo_tree_all_reduce.argtypes = [PF, C.c_int, i64, PF]
        L.tbo_ring_reduce.argtypes = [PF, C.c_int, i64, PF]
        L.tbo_row_parallel_forward.argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64, i64, i64, C.c_int, i64, PF]
        L.tbo_rmsnorm_seq.argtypes = [vp, C.c_int, i64, i64, PF, f32, PF]
        L.tbo_tree_rmsnorm.argtypes = [vp, C.c_int, i64, i64, PF, f32, PF]
        L.tbo_exp.restype = f32
        L.tbo_exp.argtypes = [f32]
        L.tbo_log.restype = f32
        L.tbo_log.argtypes = [f32]
        L.tbo_tree_logsoftmax.argtypes = [PF, i64, i64, i64, PF, PF, PI64, PF]
        L.tbo_logsoftmax_group_states.argtypes = [PF, i64, i64, i64, PF, PF]
        L.tbo_logsoftmax_chunk_states.argtypes = [PF, i64, i64, i64, PF, PF]
        L.tbo_silu_mul.argtypes = [PF, i64, i64, i64, vp, i64]
        L.tbo_residual_add.argtypes = [vp, i64, PF, i64, i64, i64]
        L.tbo_rope.argtypes = [PF, i64, i64, C.c_int, C.c_int, vp, PF, PF, vp, i64, i64]
        L.tbo_attention_prefill.argtypes = [vp, i64, vp, i64, vp, i64, i64, C.c_int, C.c_int, C.c_int,
                                            C.c_float, vp, i64]

    # -- decoder per-token kernels (numpy in/out; bf16 as uint16 bits) ---------
    def silu_mul(self, gu: np.ndarray, inter: int):
        gu = np.ascontiguousarray(gu, np.float32)
        out = np.empty((gu.shape[0], inter), np.uint16)
        _check(self.lib.tbo_silu_mul(gu.ctypes.data_as(PF), gu.shape[1], gu.shape[0], inter, _p(out), inter),
               "silu_mul")
        return out

    def residual_add(self, h: np.ndarray, f: np.ndarray):
        h = np.ascontiguousarray(h, np.uint16).copy()
        f = np.ascontiguousarray(f, np.float32)
        _check(self.lib.tbo_residual_add(_p(h), h.shape[1], f.ctypes.data_as(PF), f.shape[1], h.shape[0],
                                         h.shape[1]), "residual_add")
        return h

    def rope(self, x, col0, heads, head_dim, positions, cos_t, sin_t):
        x = np.ascontiguousarray(x, np.float32)
        pos = np.ascontiguousarray(positions, np.int32)
        c = np.ascontiguousarray(cos_t, np.float32)
        s = np.ascontiguousarray(sin_t, np.float32)
        out = np.empty((x.shape[0], heads * head_dim), np.uint16)
        _check(self.lib.tbo_rope(x.ctypes.data_as(PF), x.shape[1], col0, heads, head_dim, _p(pos),
                                 c.ctypes.data_as(PF), s.ctypes.data_as(PF), _p(out), heads * head_dim,
                                 x.shape[0]), "rope")
        return out

    def attention_prefill(self, q, k, v, batch, seq_len, nq, nkv, scale):
        q, k, v = (np.ascontiguousarray(t, np.uint16) for t in (q, k, v))
        out = np.empty((batch * seq_len, nq * 128), np.uint16)
        _check(self.lib.tbo_attention_prefill(_p(q), q.shape[1], _p(k), k.shape[1], _p(v), v.shape[1], batch,
                                              seq_len, nq, nkv, scale, _p(out), nq * 128), "attention")
        return out

    # -- inputs -------------------------------------------------------------
    def random_normal(self, seed, stream, rows, cols, dtype="bf16", mean=0.0, std=1.0):
        out = np.empty((rows, cols), np.uint16 if dtype == "bf16" else np.float32)
        _check(self.lib.tbo_random_normal(seed, stream, rows, cols, 1 if dtype == "bf16" else 0,
                                          mean, std, _p(out)), "random_normal")
        return out

    def bf16_round(self, x: float) -> int:
        return int(self.lib.tbo_bf16_round(float(x)))

    def fingerprint(self, m: np.ndarray) -> int:
        r, c = m.shape
        return int(self.lib.tbo_fingerprint(_p(m), _dt(m), r, c))

    # -- planner ------------------------------------------------------------
    def plan_blocks(self, K, block_k, k_first=0, c_max=8):
        out = (C.c_int64 * 4)()
        _check(self.lib.tbo_plan_blocks(K, block_k, k_first, c_max, out), "plan_blocks")
        return tuple(out)

    def row_shard_plan(self, K, block_k, k_first, tp, c_max):
        b = (C.c_int64 * (2 * tp))()
        _check(self.lib.tbo_make_row_shard_plan(K, block_k, k_first, tp, c_max, b), "row_shard")
        return [(b[2 * r], b[2 * r + 1]) for r in range(tp)]

    def column_shard_plan(self, N, tp):
        b = (C.c_int64 * (2 * tp))()
        _check(self.lib.tbo_make_column_shard_plan(N, tp, b), "column_shard")
        return [(b[2 * r], b[2 * r + 1]) for r in range(tp)]

    # -- kernels ------------------------------------------------------------
    def tree_reduce(self, leaves) -> float:
        v = np.ascontiguousarray(leaves, np.float32)
        o = C.c_float()
        _check(self.lib.tbo_tree_reduce(v.ctypes.data_as(PF), v.size, C.byref(o)), "tree_reduce")
        return np.float32(o.value)

    def tree_matmul(self, a, b, block_k=256, k_first=0):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.tbo_tree_matmul(_p(a), _dt(a), _p(b), _dt(b), M, K, N, block_k, k_first,
                                        out.ctypes.data_as(PF)), "tree_matmul")
        return out

    def global_tree_matmul(self, a, b, block_k=256, k_first=0, c_max=8):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.tbo_global_tree_matmul(_p(a), _dt(a), _p(b), _dt(b), M, K, N, block_k,
                                               k_first, c_max, out.ctypes.data_as(PF)),
               "global_tree_matmul")
        return out

    def tree_over_leaves(self, leaves: np.ndarray, k_first: int):
        T = leaves.shape[0]
        E = leaves[0].size
        v = np.ascontiguousarray(leaves.reshape(T, E), np.float32)
        out = np.empty(E, np.float32)
        _check(self.lib.tbo_tree_over_leaves(v.ctypes.data_as(PF), T, E, k_first,
                                             out.ctypes.data_as(PF)), "tree_over_leaves")
        return out.reshape(leaves.shape[1:])

    def sequential_matmul(self, a, b):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.tbo_sequential_matmul(_p(a), _dt(a), _p(b), _dt(b), M, K, N,
                                              out.ctypes.data_as(PF)), "sequential_matmul")
        return out

    def tree_all_reduce(self, contributions: np.ndarray):
        W = contributions.shape[0]
        c = np.ascontiguousarray(contributions, np.float32)
        out = np.empty(contributions.shape[1:], np.float32)
        _check(self.lib.tbo_tree_all_reduce(c.ctypes.data_as(PF), W, out.size,
                                            out.ctypes.data_as(PF)), "tree_all_reduce")
        return out

    def ring_reduce(self, contributions: np.ndarray):
        W = contributions.shape[0]
        c = np.ascontiguousarray(contributions, np.float32)
        out = np.empty(contributions.shape[1:], np.float32)
        _check(self.lib.tbo_ring_reduce(c.ctypes.data_as(PF), W, out.size,
                                        out.ctypes.data_as(PF)), "ring_reduce")
        return out

    def row_parallel_forward(self, a, b, tp, block_k=256, k_first=0, c_max=8):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.tbo_row_parallel_forward(_p(a), _dt(a), _p(b), _dt(b), M, K, N, block_k,
                                                 k_first, tp, c_max, out.ctypes.data_as(PF)),
               "row_parallel_forward")
        return out

    def rmsnorm_seq(self, x, gamma, eps=1e-5):
        r, c = x.shape
        g = np.ascontiguousarray(gamma, np.float32)
        out = np.empty((r, c), np.float32)
        _check(self.lib.tbo_rmsnorm_seq(_p(x), _dt(x), r, c, g.ctypes.data_as(PF), eps,
                                        out.ctypes.data_as(PF)), "rmsnorm_seq")
        return out

    def tree_rmsnorm(self, x, gamma, eps=1e-5):
        r, c = x.shape
        g = np.ascontiguousarray(gamma, np.float32)
        out = np.empty((r, c), np.float32)
        _check(self.lib.tbo_tree_rmsnorm(_p(x), _dt(x), r, c, g.ctypes.data_as(PF), eps,
                                         out.ctypes.data_as(PF)), "tree_rmsnorm")
        return out

    def exp(self, x: float) -> np.float32:
        return np.float32(self.lib.tbo_exp(float(x)))

    def log(self, x: float) -> np.float32:
        return np.float32(self.lib.tbo_log(float(x)))

    def tree_logsoftmax(self, logits, groups=8, targets=None, full=False):
        rows, V = logits.shape
        x = np.ascontiguousarray(logits, np.float32)
        lse = np.empty(rows, np.float32)
        lp = np.empty((rows, V), np.float32) if full else None
        tg = None if targets is None else np.ascontiguousarray(targets, np.int64)
        tlp = np.empty(rows, np.float32) if targets is not None else None
        _check(self.lib.tbo_tree_logsoftmax(
            x.ctypes.data_as(PF), rows, V, groups, lse.ctypes.data_as(PF),
            lp.ctypes.data_as(PF) if lp is not None else None,
            tg.ctypes.data_as(PI64) if tg is not None else None,
            tlp.ctypes.data_as(PF) if tlp is not None else None), "tree_logsoftmax")
        return lse, lp, tlp

    def logsoftmax_chunk_states(self, logits, groups=8):
        """(m, s) of every 16-logit chunk (chunks restart at each vocab group):
        rows x (groups * ceil(V / groups / 16)) each."""
        x = np.ascontiguousarray(logits, np.float32)
        rows, V = x.shape
        nc = (V // groups + 15) // 16
        m = np.empty((rows, groups * nc), np.float32)
        s = np.empty((rows, groups * nc), np.float32)
        _check(self.lib.tbo_logsoftmax_chunk_states(x.ctypes.data_as(PF), rows, V, groups, m.ctypes.data_as(PF),
                                                    s.ctypes.data_as(PF)), "chunk_states")
        return m, s

    def logsoftmax_group_states(self, logits, groups=8):
        rows, V = logits.shape
        x = np.ascontiguousarray(logits, np.float32)
        m = np.empty((rows, groups), np.float32)
        s = np.empty((rows, groups), np.float32)
        _check(self.lib.tbo_logsoftmax_group_states(x.ctypes.data_as(PF), rows, V, groups,
                                                    m.ctypes.data_as(PF), s.ctypes.data_as(PF)),
               "group_states")
        return m, s


class RefLib(_Lib):
    """The unmodified reference library (oracle/_ref/libtbik_ref.so)."""

    so_path = REF_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_plan_blocks.argtypes = [i64, PI64, i64, PI64]
        L.ref_make_row_shard_plan.argtypes = [i64, PI64, C.c_int, i64, PI64]
        L.ref_make_column_shard_plan.argtypes = [i64, C.c_int, PI64]
        L.ref_random_normal.argtypes = [u64, u64, i64, i64, C.c_int, f32, f32, vp]
        L.ref_fingerprint.restype = u64
        L.ref_fingerprint.argtypes = [vp, C.c_int, i64, i64]
        L.ref_bf16_round.restype = C.c_uint16
        L.ref_bf16_round.argtypes = [f32]
        L.ref_leaf_dot.restype = f32
        L.ref_leaf_dot.argtypes = [PF, PF, i64]
        L.ref_tree_reduce.argtypes = [PF, i64, PF]
        for fn in ("ref_tree_matmul",):
            getattr(L, fn).argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64, PI64, PF]
        L.ref_row_parallel_forward.argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64, PI64,
                                               C.c_int, i64, PF]
        L.ref_column_parallel_forward.argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64, PI64,
                                                  C.c_int, PF]
        L.ref_baseline_row_parallel_forward.argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64,
                                                        C.c_int, PF]
        L.ref_global_tree_matmul.argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64, PI64, i64, PF]
        L.ref_sequential_matmul.argtypes = [vp, C.c_int, vp, C.c_int, i64, i64, i64, PF]
        L.ref_tree_all_reduce.argtypes = [PF, C.c_int, i64, i64, PF]
        L.ref_ring_reduce.argtypes = [PF, C.c_int, i64, i64, PF]
        L.ref_device_group.argtypes = [C.c_int]
        L.ref_rmsnorm.argtypes = [vp, C.c_int, i64, i64, PF, f32, PF]
        L.ref_silu.argtypes = [vp, C.c_int, i64, i64, PF]
        L.ref_check_theorem1_exhaustive.argtypes = [C.c_int, C.c_int, C.POINTER(u64)]
        L.ref_check_collective_symmetry.argtypes = [C.c_int, i64, C.POINTER(u64)]
        L.ref_check_kernel_tp_invariance.argtypes = [C.c_int, i64, i64, i64, C.POINTER(u64)]
        L.ref_nonassoc_witness.argtypes = [PF]
        L.ref_fma_witness.argtypes = [PF]
        L.ref_leaf_order_witness.restype = u64
        L.ref_leaf_order_witness.argtypes = [PF, PF, PF]
        L.ref_matrix_write.argtypes = [C.c_char_p, vp, C.c_int, i64, i64]
        L.ref_matrix_read.argtypes = [C.c_char_p, C.POINTER(C.c_int), PI64, PI64, vp, i64]

    @staticmethod
    def _cfg(block_m, block_k, block_n, k_first):
        return (C.c_int64 * 4)(block_m, block_k, block_n, k_first)

    def set_threads(self, n: int) -> None:
        self.lib.ref_set_threads(n)

    def matrix_write(self, path, m) -> int:
        """The reference's matrix_write (matrix.cpp:211-233); returns its status (0 ok,
        1 + ErrorCode on TbikError)."""
        r, c = m.shape
        return int(self.lib.ref_matrix_write(os.fsencode(path), _p(m), _dt(m), r, c))

    def matrix_read(self, path):
        """The reference's matrix_read (matrix.cpp:235-284) -> (status, array or None)."""
        dt, r, c = C.c_int(), C.c_int64(), C.c_int64()
        st = int(self.lib.ref_matrix_read(os.fsencode(path), C.byref(dt), C.byref(r), C.byref(c), None, 0))
        if st:
            return st, None
        out = np.empty((r.value, c.value), np.float32 if dt.value == 0 else np.uint16)
        st = int(self.lib.ref_matrix_read(os.fsencode(path), C.byref(dt), C.byref(r), C.byref(c), _p(out),
                                          out.nbytes))
        return st, out

    def worker_count(self) -> int:
        return int(self.lib.ref_worker_count())

    def random_normal(self, seed, stream, rows, cols, dtype="bf16", mean=0.0, std=1.0):
        out = np.empty((rows, cols), np.uint16 if dtype == "bf16" else np.float32)
        _check(self.lib.ref_random_normal(seed, stream, rows, cols, 1 if dtype == "bf16" else 0,
                                          mean, std, _p(out)), "ref_random_normal")
        return out

    def fingerprint(self, m):
        r, c = m.shape
        return int(self.lib.ref_fingerprint(_p(m), _dt(m), r, c))

    def plan_blocks(self, K, block_k, k_first=0, c_max=8, block_m=64, block_n=128):
        out = (C.c_int64 * 4)()
        _check(self.lib.ref_plan_blocks(K, self._cfg(block_m, block_k, block_n, k_first), c_max,
                                        out), "ref_plan_blocks")
        return tuple(out)

    def row_shard_plan(self, K, block_k, k_first, tp, c_max):
        b = (C.c_int64 * (2 * tp))()
        _check(self.lib.ref_make_row_shard_plan(K, self._cfg(64, block_k, 128, k_first), tp,
                                                c_max, b), "ref_row_shard")
        return [(b[2 * r], b[2 * r + 1]) for r in range(tp)]

    def tree_matmul(self, a, b, block_k=256, k_first=0, block_m=64, block_n=128):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.ref_tree_matmul(_p(a), _dt(a), _p(b), _dt(b), M, K, N,
                                        self._cfg(block_m, block_k, block_n, k_first),
                                        out.ctypes.data_as(PF)), "ref_tree_matmul")
        return out

    def row_parallel_forward(self, a, b, tp, block_k=256, k_first=0, c_max=8, block_m=64,
                             block_n=128):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.ref_row_parallel_forward(_p(a), _dt(a), _p(b), _dt(b), M, K, N,
                                                 self._cfg(block_m, block_k, block_n, k_first),
                                                 tp, c_max, out.ctypes.data_as(PF)),
               "ref_row_parallel_forward")
        return out

    def column_parallel_forward(self, a, b, tp, block_k=256, k_first=0, block_m=64, block_n=128):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.ref_column_parallel_forward(_p(a), _dt(a), _p(b), _dt(b), M, K, N,
                                                    self._cfg(block_m, block_k, block_n, k_first),
                                                    tp, out.ctypes.data_as(PF)),
               "ref_column_parallel_forward")
        return out

    def baseline_row_parallel_forward(self, a, b, tp):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.ref_baseline_row_parallel_forward(_p(a), _dt(a), _p(b), _dt(b), M, K, N,
                                                          tp, out.ctypes.data_as(PF)),
               "ref_baseline_row_parallel_forward")
        return out

    def global_tree_matmul(self, a, b, block_k=256, k_first=0, c_max=8):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.ref_global_tree_matmul(_p(a), _dt(a), _p(b), _dt(b), M, K, N,
                                               self._cfg(64, block_k, 128, k_first), c_max,
                                               out.ctypes.data_as(PF)), "ref_global_tree_matmul")
        return out

    def sequential_matmul(self, a, b):
        M, K = a.shape
        N = b.shape[1]
        out = np.empty((M, N), np.float32)
        _check(self.lib.ref_sequential_matmul(_p(a), _dt(a), _p(b), _dt(b), M, K, N,
                                              out.ctypes.data_as(PF)), "ref_sequential_matmul")
        return out

    def tree_all_reduce(self, contributions):
        W = contributions.shape[0]
        c = np.ascontiguousarray(contributions, np.float32).reshape(W, -1)
        out = np.empty(c.shape[1], np.float32)
        _check(self.lib.ref_tree_all_reduce(c.ctypes.data_as(PF), W, 1, c.shape[1],
                                            out.ctypes.data_as(PF)), "ref_tree_all_reduce")
        return out.reshape(contributions.shape[1:])

    def ring_reduce(self, contributions):
        W = contributions.shape[0]
        c = np.ascontiguousarray(contributions, np.float32).reshape(W, -1)
        out = np.empty(c.shape[1], np.float32)
        _check(self.lib.ref_ring_reduce(c.ctypes.data_as(PF), W, 1, c.shape[1],
                                        out.ctypes.data_as(PF)), "ref_ring_reduce")
        return out.reshape(contributions.shape[1:])

    def device_group_status(self, W) -> int:
        return int(self.lib.ref_device_group(W))

    def rmsnorm(self, x, gamma, eps=1e-5):
        r, c = x.shape
        g = np.ascontiguousarray(gamma, np.float32)
        out = np.empty((r, c), np.float32)
        _check(self.lib.ref_rmsnorm(_p(x), _dt(x), r, c, g.ctypes.data_as(PF), eps,
                                    out.ctypes.data_as(PF)), "ref_rmsnorm")
        return out

    def tree_reduce(self, leaves):
        v = np.ascontiguousarray(leaves, np.float32)
        o = C.c_float()
        _check(self.lib.ref_tree_reduce(v.ctypes.data_as(PF), v.size, C.byref(o)), "ref_tree_reduce")
        return np.float32(o.value)

    def check_theorem1_exhaustive(self, max_t=6, vectors=100):
        f = C.c_uint64()
        ok = self.lib.ref_check_theorem1_exhaustive(max_t, vectors, C.byref(f))
        return bool(ok), int(f.value)

    def check_collective_symmetry(self, vectors=8, elems=8):
        d = C.c_uint64()
        ok = self.lib.ref_check_collective_symmetry(vectors, elems, C.byref(d))
        return bool(ok), int(d.value)

    def nonassoc_witness(self):
        o = (C.c_float * 7)()
        self.lib.ref_nonassoc_witness(o)
        return [np.float32(v) for v in o]

    def fma_witness(self):
        o = (C.c_float * 5)()
        self.lib.ref_fma_witness(o)
        return [np.float32(v) for v in o]

    def leaf_order_witness(self):
        a = (C.c_float * 8)()
        b = (C.c_float * 8)()
        o = (C.c_float * 2)()
        seed = self.lib.ref_leaf_order_witness(a, b, o)
        return int(seed), np.array(a, np.float32), np.array(b, np.float32), np.array(o, np.float32)


def ref_available() -> bool:
    return os.path.exists(REF_SO)
