"""Python mirror of the reference's C++ API (proj/include/tbik/*.hpp) over the C ABI.

Same names, argument meaning and error behaviour as the reference, so the
parity tests read like the reference's own checks (runner.cpp:53-214):

  reference (C++, host Matrix)                 here (torch CUDA tensors)
  -------------------------------------------  ---------------------------------------
  BlockConfig / default_block_config            BlockConfig / default_block_config
  plan_blocks (matmul.hpp:42-43)                plan_blocks
  tree_matmul (matmul.hpp:53)                   tree_matmul(a, b, cfg, leaf=...)
  DeviceGroup(int) (collective.hpp:17)          DeviceGroup(world_size)   (simulated, one GPU)
  tree_all_reduce(_per_rank), ring_reduce_...   tree_all_reduce, tree_all_reduce_per_rank,
                                                ring_reduce_baseline
  make_row/column_shard_plan (layers.hpp:27-32) make_row_shard_plan, make_column_shard_plan
  row/column_parallel_forward (layers.hpp)      row_parallel_forward, column_parallel_forward
  rmsnorm (demo.hpp:53)                         rmsnorm  (tree-ordered)
  (none: softmax_row is internal, demo.cpp:84)  log_softmax (vocab-sharded tree)
  TbikError(ErrorCode) (errors.hpp)             TbikError(ErrorCode)

Tensors: bf16 or f32, 2-D, on a CUDA device; outputs are f32 (the reference's
F32_STORED output).  Work is queued on torch's current stream.  Nothing here
falls back to the CPU.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Sequence

from ._lib import (BlockConfigC, ErrorCode, ReductionPlanC, TBIK_IPC_HANDLE_BYTES, TbikError,
                   check, lib)

F32, BF16 = 0, 1
LEAF_FMA, LEAF_TCGEN05 = 0, 1


@dataclass
class BlockConfig:
    """tbik::BlockConfig (matmul.hpp:18-25)."""
    block_m: int = 64
    block_k: int = 256
    block_n: int = 128
    k_first: int = 0

    def c(self) -> BlockConfigC:
        return BlockConfigC(self.block_m, self.block_k, self.block_n, self.k_first)


@dataclass(frozen=True)
class ReductionPlan:
    """tbik::ReductionPlan (matmul.hpp:30-35)."""
    tiles_total: int
    k_first: int
    leaves: int
    depth: int


@dataclass(frozen=True)
class ShardPlan:
    """tbik::ShardPlan (layers.hpp:17-25)."""
    mode: str  # "column" | "row"
    tp_size: int
    bounds: List[tuple]


def default_block_config(dtype: int = BF16) -> BlockConfig:
    c = BlockConfigC()
    check(lib.tbik_default_block_config(dtype, C.byref(c)))
    return BlockConfig(c.block_m, c.block_k, c.block_n, c.k_first)


def plan_blocks(K: int, cfg: BlockConfig, c_max: int) -> ReductionPlan:
    p = ReductionPlanC()
    check(lib.tbik_plan_blocks(K, C.byref(cfg.c()), c_max, C.byref(p)))
    return ReductionPlan(p.tiles_total, p.k_first, p.leaves, p.depth)


def make_row_shard_plan(k: int, cfg: BlockConfig, tp_size: int, c_max: int) -> ShardPlan:
    b = (C.c_int64 * (2 * max(tp_size, 1)))()
    check(lib.tbik_make_row_shard_plan(k, C.byref(cfg.c()), tp_size, c_max, b))
    return ShardPlan("row", tp_size, [(b[2 * r], b[2 * r + 1]) for r in range(tp_size)])


def make_column_shard_plan(n: int, tp_size: int) -> ShardPlan:
    b = (C.c_int64 * (2 * max(tp_size, 1)))()
    check(lib.tbik_make_column_shard_plan(n, tp_size, b))
    return ShardPlan("column", tp_size, [(b[2 * r], b[2 * r + 1]) for r in range(tp_size)])


def device_available() -> bool:
    return bool(lib.tbik_device_available())


def launch_count() -> int:
    """Kernels launched by libtbik_b200 so far in this process."""
    return int(lib.tbik_launch_count())


def last_kernel() -> str:
    """tbik_last_kernel: the last tree-GEMM kernel this thread launched."""
    return lib.tbik_last_kernel().decode()


SCHEDULE_KNOBS = ("tc_pair", "tc_abox", "tc_group_m", "tc_units", "tc_deep", "tc_acc4", "tc_skinny", "sk_mt",
                  "sk_units", "sk_leaf", "sk_bn", "fma_v1", "group_fused", "group_overlap", "ar_two_phase_bytes",
                  "tc_wide", "tc_wide_tail", "sk_ks", "sk_pdl", "sk_trace", "sk_pair", "attn_sv1", "attn_tc5", "tc_pdl")


def set_schedule(name, value: int = -1) -> None:
    """tbik_set_schedule: override one launch-schedule choice (value < 0 unsets;
    name None clears all).  Schedules never change bits -- the tests prove it."""
    check(lib.tbik_set_schedule(name.encode() if name is not None else None, int(value)))


@contextlib.contextmanager
def schedule(**knobs):
    """with schedule(tc_pair=0, sk_units=2): ... -- overrides inside, all cleared after."""
    set_schedule(None)
    try:
        for k, v in knobs.items():
            set_schedule(k, v)
        yield
    finally:
        set_schedule(None)


# ---- tensor helpers -----------------------------------------------------------------
def _torch():
    import torch
    return torch


def _dt(t) -> int:
    torch = _torch()
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise TbikError(ErrorCode.UnknownDtype, f"unsupported dtype {t.dtype}")


def _mat(t, name: str):
    if t.dim() != 2:
        raise TbikError(ErrorCode.BadDimension, f"{name} must be 2-D")
    if not t.is_cuda:
        raise TbikError(ErrorCode.NoDevice, f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.stride(1) != 1:
        raise TbikError(ErrorCode.BadArgument, f"{name} must be row-major (unit column stride)")
    return C.c_void_p(t.data_ptr()), _dt(t), t.stride(0)


def _stream():
    return C.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _empty_f32(rows, cols, like):
    return _torch().empty((rows, cols), dtype=_torch().float32, device=like.device)


# ---- the TBIK GEMM --------------------------------------------------------------------
def tree_matmul(a, b, cfg: BlockConfig | None = None, leaf: int = LEAF_TCGEN05, out=None):
    """tree_matmul (matmul.hpp:53): C = A x B with the tree reduction over K; f32 out."""
    cfg = cfg or default_block_config(BF16)
    if a.shape[1] != b.shape[0]:
        raise TbikError(ErrorCode.ShapeMismatch,
                        f"tree_matmul: inner dimensions differ, {a.shape[1]} vs {b.shape[0]}")
    M, K = a.shape
    N = b.shape[1]
    pa, da, lda = _mat(a, "A")
    pb, db, ldb = _mat(b, "B")
    out = _empty_f32(M, N, a) if out is None else out
    pc, _, ldc = _mat(out, "C")
    check(lib.tbik_tree_matmul(pa, da, lda, pb, db, ldb, pc, ldc, M, N, K, C.byref(cfg.c()), leaf,
                               _stream()))
    return out


def tree_matmul_hostio(a_host, b, cfg: BlockConfig | None = None, leaf: int = LEAF_TCGEN05, out=None,
                       chunk_rows: int = 0):
    """tree_matmul with HOST activations and a HOST f32 result (weights `b` on the
    device): H2D, GEMM and D2H overlap over row chunks (tbik_tree_matmul_hostio).
    Asynchronous on the current stream like every other entry point."""
    torch = _torch()
    cfg = cfg or default_block_config(_dt(a_host))
    M, K = a_host.shape
    N = b.shape[1]
    if a_host.is_cuda or not b.is_cuda:
        raise TbikError(ErrorCode.BadArgument, "tree_matmul_hostio: A must be a host tensor, B a device tensor")
    if a_host.stride(1) != 1 or b.stride(1) != 1:
        raise TbikError(ErrorCode.BadArgument, "tree_matmul_hostio: row-major operands required")
    out = torch.empty((M, N), dtype=torch.float32, pin_memory=True) if out is None else out
    if out.is_cuda or out.dtype != torch.float32 or out.stride(1) != 1:
        raise TbikError(ErrorCode.BadArgument, "tree_matmul_hostio: out must be a host f32 row-major tensor")
    check(lib.tbik_tree_matmul_hostio(C.c_void_p(a_host.data_ptr()), _dt(a_host), a_host.stride(0),
                                      C.c_void_p(b.data_ptr()), _dt(b), b.stride(0), C.c_void_p(out.data_ptr()),
                                      out.stride(0), M, N, K, C.byref(cfg.c()), leaf, chunk_rows, _stream()))
    return out


def tree_matmul_leaves(a, b, cfg: BlockConfig | None = None, leaf: int = LEAF_TCGEN05):
    """Every leaf partial product P_t as leaves[t] (M x N f32) -- verification entry."""
    cfg = cfg or default_block_config(BF16)
    M, K = a.shape
    N = b.shape[1]
    T = plan_blocks(K, cfg, 1).tiles_total
    out = _torch().empty((T, M, N), dtype=_torch().float32, device=a.device)
    pa, da, lda = _mat(a, "A")
    pb, db, ldb = _mat(b, "B")
    check(lib.tbik_tree_matmul_leaves(pa, da, lda, pb, db, ldb, C.c_void_p(out.data_ptr()), M, N, K,
                                      C.byref(cfg.c()), leaf, _stream()))
    return out


class DeviceGroup:
    """tbik::DeviceGroup (collective.hpp:15-23): `world_size` simulated ranks on
    the current GPU, exactly like the reference's in-process group."""

    def __init__(self, world_size: int):
        if world_size < 1 or world_size & (world_size - 1):
            raise TbikError(ErrorCode.BadWorldSize,
                            f"world size must be a power of two, got {world_size}")
        self._w = world_size

    def world_size(self) -> int:
        return self._w


def _ptr_array(ts: Sequence):
    arr = (C.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr()
    return arr


def _require_uniform(group: DeviceGroup, xs: Sequence) -> None:
    """require_uniform (collective.cpp:20-36)."""
    if len(xs) != group.world_size():
        raise TbikError(ErrorCode.CollectiveMismatch,
                        f"expected {group.world_size()} contributions, got {len(xs)}")
    for r, x in enumerate(xs[1:], 1):
        if x.shape != xs[0].shape or x.dtype != xs[0].dtype:
            raise TbikError(ErrorCode.CollectiveMismatch,
                            f"rank {r} contribution shape/dtype differs")


def all_gather(group: DeviceGroup, xs: Sequence) -> list:
    """all_gather (collective.cpp:46-50): the rank-indexed list, unchanged."""
    _require_uniform(group, xs)
    return list(xs)


def tree_all_reduce(group: DeviceGroup, xs: Sequence):
    """tree_all_reduce (collective.hpp:38-39): Algorithm-2 order, f32 only."""
    _require_uniform(group, xs)
    torch = _torch()
    if xs[0].dtype != torch.float32:
        raise TbikError(ErrorCode.CollectiveMismatch, "tree_all_reduce expects f32 inputs")
    xs = [x.contiguous() for x in xs]
    out = torch.empty_like(xs[0])
    check(lib.tbik_tree_all_reduce_local(_ptr_array(xs), len(xs), C.c_void_p(out.data_ptr()),
                                         out.numel(), _stream()))
    return out


def tree_all_reduce_per_rank(group: DeviceGroup, xs: Sequence) -> list:
    """tree_all_reduce_per_rank (collective.hpp:33-34): every simulated rank
    reduces its own gathered copy; results are checked rank-symmetric
    (collective.cpp:79-85) and CollectiveMismatch is raised otherwise."""
    outs = [tree_all_reduce(group, xs) for _ in range(group.world_size())]
    torch = _torch()
    for r in range(1, len(outs)):
        if not torch.equal(outs[0].view(torch.int32), outs[r].view(torch.int32)):
            raise TbikError(ErrorCode.CollectiveMismatch,
                            f"tree_all_reduce produced rank-divergent results at rank {r}")
    return outs


def ring_reduce_baseline(group: DeviceGroup, xs: Sequence):
    """ring_reduce_baseline (collective.hpp:43-44): labelled non-invariant stand-in."""
    _require_uniform(group, xs)
    xs = [x.contiguous() for x in xs]
    out = _torch().empty_like(xs[0])
    check(lib.tbik_ring_reduce_local(_ptr_array(xs), len(xs), C.c_void_p(out.data_ptr()),
                                     out.numel(), _stream()))
    return out


def row_parallel_forward(x, w, group: DeviceGroup, cfg: BlockConfig | None = None, c_max: int = 8,
                         leaf: int = LEAF_TCGEN05, out=None):
    """row_parallel_forward (layers.hpp:43-45) with simulated ranks on one GPU."""
    cfg = cfg or default_block_config(BF16)
    if x.shape[1] != w.shape[0]:
        raise TbikError(ErrorCode.ShapeMismatch, "row_parallel_forward: inner dimensions differ")
    M, K = x.shape
    N = w.shape[1]
    px, dx, ldx = _mat(x, "X")
    pw, dw, ldw = _mat(w, "W")
    out = _empty_f32(M, N, x) if out is None else out
    py, _, ldy = _mat(out, "Y")
    check(lib.tbik_row_parallel_forward_local(px, dx, ldx, pw, dw, ldw, py, ldy, M, N, K,
                                              group.world_size(), C.byref(cfg.c()), c_max, leaf,
                                              _stream()))
    return out


def column_parallel_forward(x, w, group: DeviceGroup, cfg: BlockConfig | None = None,
                            leaf: int = LEAF_TCGEN05, out=None):
    """column_parallel_forward (layers.hpp:36-38) with simulated ranks on one GPU."""
    cfg = cfg or default_block_config(BF16)
    if x.shape[1] != w.shape[0]:
        raise TbikError(ErrorCode.ShapeMismatch, "column_parallel_forward: inner dimensions differ")
    M, K = x.shape
    N = w.shape[1]
    px, dx, ldx = _mat(x, "X")
    pw, dw, ldw = _mat(w, "W")
    out = _empty_f32(M, N, x) if out is None else out
    py, _, ldy = _mat(out, "Y")
    check(lib.tbik_column_parallel_forward_local(px, dx, ldx, pw, dw, ldw, py, ldy, M, N, K,
                                                 group.world_size(), C.byref(cfg.c()), leaf,
                                                 _stream()))
    return out


def interleave_gate_up(w):
    """[gate | up] (K x 2I) -> columns interleaved gate_0, up_0, gate_1, up_1, ... --
    the B layout of tree_matmul_silu_mul (a pure column permutation: each column's
    tree GEMM is unchanged)."""
    K, N2 = w.shape
    inter = N2 // 2
    return w.view(K, 2, inter).transpose(1, 2).reshape(K, N2).contiguous()


def tree_matmul_silu_mul(x, w_il, group: DeviceGroup | None = None, cfg: BlockConfig | None = None,
                         leaf: int = LEAF_TCGEN05, out=None):
    """bf16(silu(x @ W_gate) * (x @ W_up)) with W's columns interleaved (interleave_gate_up),
    column-parallel over `group`'s simulated ranks: rank r owns gate/up pairs
    [r I/tp, (r+1) I/tp) (layers.cpp:48-72).  SiLU*up runs in the GEMM epilogue."""
    torch = _torch()
    cfg = cfg or default_block_config(BF16)
    tp = group.world_size() if group is not None else 1
    M, K = x.shape
    N2 = w_il.shape[1]
    inter = N2 // 2
    if w_il.shape[0] != K or N2 % 2 or inter % tp:
        raise TbikError(ErrorCode.ShapeMismatch, "tree_matmul_silu_mul: bad shapes")
    out = torch.empty((M, inter), dtype=torch.bfloat16, device=x.device) if out is None else out
    px, dx, ldx = _mat(x, "X")
    _, dw, ldw = _mat(w_il, "W")
    ir = inter // tp
    for r in range(tp):
        pw = C.c_void_p(w_il.data_ptr() + 2 * ir * r * w_il.element_size())
        po = C.c_void_p(out.data_ptr() + ir * r * out.element_size())
        check(lib.tbik_tree_matmul_silu_mul(px, dx, ldx, pw, dw, ldw, po, out.stride(0), M, ir, K,
                                            C.byref(cfg.c()), leaf, _stream()))
    return out


# ---- one process, several GPUs ------------------------------------------------------------
class LocalGroup:
    """The reference's DeviceGroup held by ONE process with rank r on GPU
    device_ids[r] (tbik_local_group_*): per-rank streams, peer access, and the
    row-parallel forward whose partials meet over peer memory on rank 0's GPU."""

    def __init__(self, device_ids: Sequence[int]):
        W = len(device_ids)
        ids = (C.c_int * W)(*device_ids)
        h = C.c_void_p()
        check(lib.tbik_local_group_create(W, ids, C.byref(h)))
        self._h, self.world, self.devices = h, W, list(device_ids)

    def close(self) -> None:
        if self._h:
            lib.tbik_local_group_destroy(self._h)
            self._h = None

    def row_parallel_forward(self, x_shards: Sequence, w_shards: Sequence, K_global: int,
                             cfg: BlockConfig | None = None, c_max: int = 8, leaf: int = LEAF_TCGEN05, out=None):
        """x_shards[r] / w_shards[r]: rank r's make_row_shard_plan range, on devices[r]."""
        torch = _torch()
        cfg = cfg or default_block_config(BF16)
        W = self.world
        M, N = x_shards[0].shape[0], w_shards[0].shape[1]
        xs = (C.c_void_p * W)(*[t.data_ptr() for t in x_shards])
        ws = (C.c_void_p * W)(*[t.data_ptr() for t in w_shards])
        ldx = (C.c_int64 * W)(*[t.stride(0) for t in x_shards])
        ldw = (C.c_int64 * W)(*[t.stride(0) for t in w_shards])
        out = torch.empty((M, N), dtype=torch.float32, device=f"cuda:{self.devices[0]}") if out is None else out
        torch.cuda.synchronize()  # inputs complete on every device (the ABI orders only rank 0's stream)
        check(lib.tbik_local_group_row_parallel_forward(self._h, xs, _dt(x_shards[0]), ldx, ws, _dt(w_shards[0]), ldw,
                                                        C.c_void_p(out.data_ptr()), out.stride(0), M, N, K_global,
                                                        C.byref(cfg.c()), c_max, leaf, _stream()))
        return out


# ---- the labelled non-invariant status quo ----------------------------------------------
def baseline_row_parallel_forward(x, w, group: DeviceGroup):
    """baseline_row_parallel_forward (layers.hpp:48-49): cuBLAS per K/tp shard + ring sum."""
    M, K = x.shape
    N = w.shape[1]
    px, dx, ldx = _mat(x, "X")
    pw, dw, ldw = _mat(w, "W")
    out = _empty_f32(M, N, x)
    check(lib.tbik_baseline_row_parallel_forward_local(px, dx, ldx, pw, dw, ldw, C.c_void_p(out.data_ptr()), N,
                                                       M, N, K, group.world_size(), _stream()))
    return out


def baseline_column_parallel_forward(x, w, group: DeviceGroup):
    """baseline_column_parallel_forward (layers.hpp:53-54): cuBLAS per column shard."""
    M, K = x.shape
    N = w.shape[1]
    px, dx, ldx = _mat(x, "X")
    pw, dw, ldw = _mat(w, "W")
    out = _empty_f32(M, N, x)
    check(lib.tbik_baseline_column_parallel_forward_local(px, dx, ldx, pw, dw, ldw, C.c_void_p(out.data_ptr()), N,
                                                          M, N, K, group.world_size(), _stream()))
    return out


def silu(x):
    """silu (demo.hpp:56): z / (1 + exp(-z)) in f32 (the library's exp)."""
    rows, cols = x.shape
    px, dx, ldx = _mat(x, "x")
    out = _empty_f32(rows, cols, x)
    check(lib.tbik_silu(px, dx, ldx, rows, cols, C.c_void_p(out.data_ptr()), cols, _stream()))
    return out


def leaf_dot(a, b):
    """leaf_dot (matmul.hpp:48) of two f32 device vectors: ascending fma from +0."""
    torch = _torch()
    out = torch.empty(1, dtype=torch.float32, device=a.device)
    check(lib.tbik_leaf_dot(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), a.numel(),
                            C.c_void_p(out.data_ptr()), _stream()))
    return out


# ---- tree-ordered reductions ----------------------------------------------------------
def rmsnorm(x, gamma, eps: float = 1e-5, out_dtype=None):
    """rmsnorm (demo.hpp:53) with the canonical tree sum of squares."""
    torch = _torch()
    rows, cols = x.shape
    if gamma.numel() != cols:
        raise TbikError(ErrorCode.ShapeMismatch, f"rmsnorm: gamma length {gamma.numel()} != cols {cols}")
    out_dtype = out_dtype or torch.float32
    out = torch.empty((rows, cols), dtype=out_dtype, device=x.device)
    px, dx, ldx = _mat(x, "X")
    g = gamma.to(torch.float32).contiguous()
    check(lib.tbik_tree_rmsnorm(px, dx, ldx, C.c_void_p(g.data_ptr()), eps, C.c_void_p(out.data_ptr()),
                                _dt(out), out.stride(0), rows, cols, _stream()))
    return out


def chunk_states_per_row(V: int, groups: int) -> int:
    """(m, s) chunk states per row of a V-wide logit block cut into `groups` vocab
    groups: 16-logit chunks, restarting at every group."""
    return groups * ((V // groups + 15) // 16)


def tree_matmul_logits(a, w, groups: int, cfg: BlockConfig | None = None, leaf: int = LEAF_TCGEN05, out=None,
                       chunks=None):
    """The lm_head with the log-softmax's first pass fused (tbik_tree_matmul_logits):
    returns (logits [M, N] f32, chunk states [M, states, 2] f32) -- the states come
    from the tcgen05 GEMM's epilogue when it is one FULL launch, else from a pass
    over the logits (same bits)."""
    torch = _torch()
    cfg = cfg or default_block_config(BF16)
    M, K = a.shape
    N = w.shape[1]
    pa, da, lda = _mat(a, "A")
    pw, dw, ldw = _mat(w, "W")
    out = _empty_f32(M, N, a) if out is None else out
    pc, _, ldc = _mat(out, "C")
    nst = chunk_states_per_row(N, groups)
    chunks = torch.empty((M, nst, 2), dtype=torch.float32, device=a.device) if chunks is None else chunks
    check(lib.tbik_tree_matmul_logits(pa, da, lda, pw, dw, ldw, pc, ldc, C.c_void_p(chunks.data_ptr()),
                                      chunks.stride(0) // 2, M, N, K, groups, C.byref(cfg.c()), leaf, _stream()))
    return out, chunks


def column_parallel_logits(x, w, group: DeviceGroup, groups: int, cfg: BlockConfig | None = None,
                           leaf: int = LEAF_TCGEN05):
    """column_parallel_forward of the lm_head (layers.cpp:48-72) with the fused chunk
    states: simulated rank r owns vocab columns [r V/tp, (r+1) V/tp) = groups
    [r G/tp, (r+1) G/tp); its logits and chunk states land at their offsets."""
    torch = _torch()
    tp = group.world_size()
    M = x.shape[0]
    V = w.shape[1]
    if V % tp or groups % tp:
        raise TbikError(ErrorCode.ShardError, "lm_head: vocab / groups not divisible by tp")
    vl, gl = V // tp, groups // tp
    logits = torch.empty((M, V), dtype=torch.float32, device=x.device)
    nst = chunk_states_per_row(V, groups)
    chunks = torch.empty((M, nst, 2), dtype=torch.float32, device=x.device)
    ns = chunk_states_per_row(vl, gl)
    for r in range(tp):
        tree_matmul_logits(x, w[:, r * vl:(r + 1) * vl], gl, cfg, leaf, out=logits[:, r * vl:(r + 1) * vl],
                           chunks=chunks[:, r * ns:(r + 1) * ns])
    return logits, chunks


def _finish(logits, lse, v_offset, targets, full, lp, tlp):
    pl, _, ld = _mat(logits, "logits")
    rows, vl = logits.shape
    if lp is not None or tlp is not None:
        check(lib.tbik_logsoftmax_finish(pl, ld, rows, vl, C.c_void_p(lse.data_ptr()),
                                         C.c_void_p(lp.data_ptr()) if lp is not None else None,
                                         lp.stride(0) if lp is not None else vl,
                                         C.c_void_p(targets.data_ptr()) if targets is not None else None, v_offset,
                                         C.c_void_p(tlp.data_ptr()) if tlp is not None else None, _stream()))


def log_softmax(logits, groups: int = 8, tp: int = 1, targets=None, full: bool = True, chunks=None):
    """Vocab-sharded tree log-softmax over `tp` simulated shards.
    Returns (lse[rows], logprobs[rows, V] or None, target_logprobs[rows] or None).
    `chunks`: the logits' 16-column (m, s) chunk states (tree_matmul_logits /
    column_parallel_logits) -- then the first pass does not re-read the logits."""
    torch = _torch()
    rows, V = logits.shape
    pl, dl, ld = _mat(logits, "logits")
    if dl != F32:
        raise TbikError(ErrorCode.UnknownDtype, "log_softmax expects f32 logits")
    if chunks is not None:
        if tp < 1 or tp & (tp - 1) or V % tp or groups % tp:
            raise TbikError(ErrorCode.ShardError, "log_softmax: vocab / groups not divisible by tp")
        vl, gl = V // tp, groups // tp
        ns = chunk_states_per_row(vl, gl)
        ms = torch.empty((tp, rows, 2), dtype=torch.float32, device=logits.device)
        for r in range(tp):
            check(lib.tbik_logsoftmax_shard_state_chunks(C.c_void_p(chunks[:, r * ns:].data_ptr()),
                                                         chunks.stride(0) // 2, rows, vl, gl,
                                                         C.c_void_p(ms[r].data_ptr()), _stream()))
        lse = torch.empty(rows, dtype=torch.float32, device=logits.device)
        check(lib.tbik_logsoftmax_merge(_ptr_array([ms[r] for r in range(tp)]), tp, rows,
                                        C.c_void_p(lse.data_ptr()), _stream()))
        lp = torch.empty((rows, V), dtype=torch.float32, device=logits.device) if full else None
        tg = tlp = None
        if targets is not None:
            tg = targets.to(torch.int64).contiguous()
            tlp = torch.empty(rows, dtype=torch.float32, device=logits.device)
        for r in range(tp):
            _finish(logits[:, r * vl:(r + 1) * vl], lse, r * vl, tg, full,
                    lp[:, r * vl:(r + 1) * vl] if lp is not None else None, tlp)
        return lse, lp, tlp
    lse = torch.empty(rows, dtype=torch.float32, device=logits.device)
    lp = torch.empty((rows, V), dtype=torch.float32, device=logits.device) if full else None
    tlp = None
    tg = None
    if targets is not None:
        tg = targets.to(torch.int64).contiguous()
        tlp = torch.empty(rows, dtype=torch.float32, device=logits.device)
    check(lib.tbik_tree_logsoftmax_local(
        pl, ld, rows, V, groups, tp, C.c_void_p(lse.data_ptr()),
        C.c_void_p(lp.data_ptr()) if lp is not None else None, V,
        C.c_void_p(tg.data_ptr()) if tg is not None else None,
        C.c_void_p(tlp.data_ptr()) if tlp is not None else None, _stream()))
    return lse, lp, tlp


# ---- the reference's TBIK matrix file -------------------------------------------------
def matrix_write(path: str, m) -> None:
    """matrix_write (matrix.hpp:86): m is a host (CPU) f32 or bf16 2-D tensor."""
    torch = _torch()
    if m.is_cuda:
        raise TbikError(ErrorCode.BadArgument, "matrix_write: host tensor expected")
    if m.dim() != 2 or m.dtype not in (torch.float32, torch.bfloat16):
        raise TbikError(ErrorCode.UnknownDtype, "matrix_write: 2-D f32 or bf16 tensor expected")
    c = m.contiguous()
    check(lib.tbik_matrix_write(os.fsencode(path), C.c_void_p(c.data_ptr()), _dt(c), c.shape[0], c.shape[1]))


def matrix_read(path: str):
    """matrix_read (matrix.hpp:87): returns a host f32 or bf16 tensor."""
    torch = _torch()
    dt, rows, cols = C.c_int(), C.c_int64(), C.c_int64()
    check(lib.tbik_matrix_read_header(os.fsencode(path), C.byref(dt), C.byref(rows), C.byref(cols)))
    out = torch.empty((rows.value, cols.value), dtype=torch.float32 if dt.value == F32 else torch.bfloat16)
    nbytes = out.numel() * out.element_size()
    buf = out if nbytes else torch.empty(1, dtype=torch.uint8)
    check(lib.tbik_matrix_read(os.fsencode(path), C.c_void_p(buf.data_ptr()), max(nbytes, 1)))
    return out


def sync() -> None:
    check(lib.tbik_sync(_stream()))


# ---- one process per GPU ----------------------------------------------------------------
class PeerGroup:
    """DeviceGroup whose ranks are processes (one per GPU) joined over NVLink peer
    memory.  Handles are exchanged with torch.distributed (any backend: gloo
    works for the exchange; the data path never touches it)."""

    def __init__(self, world_size: int, rank: int, device: int, capacity_elems: int, dist=None):
        h = C.c_void_p()
        check(lib.tbik_group_create(world_size, rank, device, capacity_elems, C.byref(h)))
        self._h = h
        self.world = world_size
        self.rank = rank
        mine = (C.c_char * TBIK_IPC_HANDLE_BYTES)()
        check(lib.tbik_group_ipc_handle(h, mine))
        handles = exchange_handles(bytes(mine), world_size, dist)
        blob = (C.c_char * (TBIK_IPC_HANDLE_BYTES * world_size)).from_buffer_copy(b"".join(handles))
        check(lib.tbik_group_open_peers(h, blob))

    def close(self) -> None:
        if self._h:
            lib.tbik_group_destroy(self._h)
            self._h = None

    def fused_count(self) -> int:
        """Row-parallel forwards that ran as one fused GEMM + tree all-reduce kernel."""
        return int(lib.tbik_group_fused_count(self._h))

    def tree_all_reduce(self, partial, out=None):
        torch = _torch()
        out = torch.empty_like(partial) if out is None else out
        check(lib.tbik_group_tree_all_reduce(self._h, C.c_void_p(partial.data_ptr()),
                                             C.c_void_p(out.data_ptr()), partial.numel(), _stream()))
        return out

    def barrier(self) -> None:
        """Device-side barrier over the group (stream-ordered)."""
        check(lib.tbik_group_barrier(self._h, _stream()))

    def all_gather(self, local, out=None):
        """all_gather as the column-parallel concatenation (layers.cpp:61-70): rank q's
        [rows x cols] block (bf16 or f32) -> columns [q*cols, (q+1)*cols) of
        out [rows x W*cols] on every rank."""
        torch = _torch()
        p, _, ld = _mat(local, "local")
        rows, cols = local.shape
        out = torch.empty((rows, cols * self.world), dtype=local.dtype, device=local.device) if out is None else out
        if out.dtype != local.dtype or out.shape[0] != rows or out.shape[1] < cols * self.world:
            raise TbikError(ErrorCode.ShapeMismatch, "all_gather: out must be [rows, W*cols] of the same dtype")
        po, _, ldo = _mat(out, "out")
        check(lib.tbik_group_all_gather(self._h, p, rows, cols, ld, local.element_size(), po, ldo, _stream()))
        return out

    def log_softmax(self, logits_shard, groups_local: int, v_offset: int, targets=None, full: bool = True,
                    chunks=None):
        """Vocab-sharded tree log-softmax over the group: this rank's logits
        [rows x V/W] (its column shard of the vocabulary, `groups_local` = G/W of the
        canonical vocab groups) -> (lse[rows] identical on every rank, this rank's
        log-prob columns or None, target log-probs of the targets in this shard or
        None).  8 bytes per row cross ranks; bit-identical to log_softmax(tp=W)."""
        torch = _torch()
        rows, vl = logits_shard.shape
        pl, dl, ld = _mat(logits_shard, "logits")
        if dl != F32:
            raise TbikError(ErrorCode.UnknownDtype, "log_softmax expects f32 logits")
        dev = logits_shard.device
        ms = torch.empty((rows, 2), dtype=torch.float32, device=dev)
        if chunks is not None:  # the lm_head epilogue's chunk states: the logits are not re-read
            check(lib.tbik_logsoftmax_shard_state_chunks(C.c_void_p(chunks.data_ptr()), chunks.stride(0) // 2, rows, vl,
                                                         groups_local, C.c_void_p(ms.data_ptr()), _stream()))
        else:
            check(lib.tbik_logsoftmax_shard_state(pl, ld, rows, vl, groups_local, C.c_void_p(ms.data_ptr()),
                                                  _stream()))
        lse = torch.empty(rows, dtype=torch.float32, device=dev)
        check(lib.tbik_group_logsoftmax_merge(self._h, C.c_void_p(ms.data_ptr()), rows, C.c_void_p(lse.data_ptr()),
                                              _stream()))
        lp = torch.empty((rows, vl), dtype=torch.float32, device=dev) if full else None
        tlp = tg = None
        if targets is not None:
            tg = targets.to(torch.int64).contiguous()
            tlp = torch.full((rows,), float("nan"), dtype=torch.float32, device=dev)
        if lp is not None or tlp is not None:
            check(lib.tbik_logsoftmax_finish(pl, ld, rows, vl, C.c_void_p(lse.data_ptr()),
                                             C.c_void_p(lp.data_ptr()) if lp is not None else None, vl,
                                             C.c_void_p(tg.data_ptr()) if tg is not None else None, v_offset,
                                             C.c_void_p(tlp.data_ptr()) if tlp is not None else None, _stream()))
        return lse, lp, tlp

    def row_parallel_forward(self, x_shard, w_shard, K_global: int, cfg: BlockConfig | None = None,
                             c_max: int = 8, leaf: int = LEAF_TCGEN05, out=None):
        cfg = cfg or default_block_config(BF16)
        M = x_shard.shape[0]
        N = w_shard.shape[1]
        px, dx, ldx = _mat(x_shard, "X")
        pw, dw, ldw = _mat(w_shard, "W")
        out = _empty_f32(M, N, x_shard) if out is None else out
        check(lib.tbik_group_row_parallel_forward(self._h, px, dx, ldx, pw, dw, ldw,
                                                  C.c_void_p(out.data_ptr()), N, M, N, K_global,
                                                  C.byref(cfg.c()), c_max, leaf, _stream()))
        return out


def _group_row_parallel_hostio(self, x_host_shard, w_shard, K_global: int, cfg: BlockConfig | None = None,
                               c_max: int = 8, leaf: int = LEAF_TCGEN05, out=None, chunk_rows: int = 0):
    """PeerGroup.row_parallel_forward with this rank's HOST X shard and a HOST f32
    result (tbik_group_row_parallel_forward_hostio)."""
    torch = _torch()
    cfg = cfg or default_block_config(BF16)
    M, Kr = x_host_shard.shape
    N = w_shard.shape[1]
    out = torch.empty((M, N), dtype=torch.float32, pin_memory=True) if out is None else out
    check(lib.tbik_group_row_parallel_forward_hostio(
        self._h, C.c_void_p(x_host_shard.data_ptr()), _dt(x_host_shard), x_host_shard.stride(0),
        C.c_void_p(w_shard.data_ptr()), _dt(w_shard), w_shard.stride(0), C.c_void_p(out.data_ptr()), out.stride(0),
        M, N, Kr, K_global, C.byref(cfg.c()), c_max, leaf, chunk_rows, _stream()))
    return out


PeerGroup.row_parallel_forward_hostio = _group_row_parallel_hostio


def exchange_handles(mine: bytes, world_size: int, dist=None) -> list:
    """Rank-indexed all-gather of the fixed-size IPC handle blobs (host metadata
    only).  Pure function of the inputs: the result is ordered by rank, never by
    arrival (collective.cpp:46-50)."""
    if world_size == 1:
        return [mine]
    if dist is None:
        import torch.distributed as dist  # noqa: F811
    gathered: list = [None] * world_size
    dist.all_gather_object(gathered, mine)
    for r, blob in enumerate(gathered):
        if not isinstance(blob, (bytes, bytearray)) or len(blob) != TBIK_IPC_HANDLE_BYTES:
            raise TbikError(ErrorCode.CollectiveMismatch, f"bad handle blob from rank {r}")
    return [bytes(b) for b in gathered]
