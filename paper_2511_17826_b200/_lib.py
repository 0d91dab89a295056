"""ctypes binding of libtbik_b200.so (the C ABI declared in include/tbik_b200.h).

The library is built in-tree (paper_2511_17826_b200/csrc/Makefile, driven by
__graft_entry__.build()).  There is deliberately no fallback: if the shared
object is missing this module raises at import, and every compute entry point
returns TBIK_NO_DEVICE (-> TbikError) when no sm_100 GPU is visible.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtbik_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "tbik_b200.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for the TBIK kernels)")

lib = C.CDLL(LIB_PATH)


class ErrorCode(enum.IntEnum):
    """tbik::ErrorCode (errors.hpp:8-20), offset by one, plus device codes."""
    BadDimension = 1
    ShapeMismatch = 2
    BadMagic = 3
    Truncated = 4
    UnknownDtype = 5
    PlanInfeasible = 6
    ShardError = 7
    BadWorldSize = 8
    CollectiveMismatch = 9
    BadArgument = 10
    Io = 11
    CudaError = 100
    NoDevice = 101
    Unsupported = 102


class TbikError(RuntimeError):
    """Mirror of tbik::TbikError (errors.hpp:22-31): carries an ErrorCode."""

    def __init__(self, code: int, what: str):
        try:
            self.code = ErrorCode(code)
        except ValueError:
            self.code = code
        super().__init__(f"{getattr(self.code, 'name', code)}: {what}")


def check(status: int) -> None:
    if status != 0:
        raise TbikError(status, lib.tbik_last_error().decode(errors="replace"))


class BlockConfigC(C.Structure):
    _fields_ = [("block_m", C.c_int64), ("block_k", C.c_int64), ("block_n", C.c_int64),
                ("k_first", C.c_int64)]


class ReductionPlanC(C.Structure):
    _fields_ = [("tiles_total", C.c_int64), ("k_first", C.c_int64), ("leaves", C.c_int64),
                ("depth", C.c_int64)]


i64, vp, ci = C.c_int64, C.c_void_p, C.c_int
PCFG = C.POINTER(BlockConfigC)
PI64 = C.POINTER(C.c_int64)
PF = C.c_void_p

_SIGS = {
    "tbik_status_string": (C.c_char_p, [ci]),
    "tbik_last_error": (C.c_char_p, []),
    "tbik_version": (ci, []),
    "tbik_device_available": (ci, []),
    "tbik_sync": (ci, [vp]),
    "tbik_launch_count": (C.c_uint64, []),
    "tbik_last_kernel": (C.c_char_p, []),
    "tbik_set_schedule": (ci, [C.c_char_p, i64]),
    "tbik_default_block_config": (ci, [ci, PCFG]),
    "tbik_plan_blocks": (ci, [i64, PCFG, i64, C.POINTER(ReductionPlanC)]),
    "tbik_make_row_shard_plan": (ci, [i64, PCFG, ci, i64, PI64]),
    "tbik_make_column_shard_plan": (ci, [i64, ci, PI64]),
    "tbik_tree_matmul": (ci, [vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, i64, PCFG, ci, vp]),
    "tbik_tree_matmul_leaves": (ci, [vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, PCFG, ci, vp]),
    "tbik_tree_matmul_silu_mul": (ci, [vp, ci, i64, vp, ci, i64, vp, i64, i64, i64, i64, PCFG, ci, vp]),
    "tbik_column_parallel_forward_local": (ci, [vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, i64, ci,
                                                PCFG, ci, vp]),
    "tbik_row_parallel_forward_local": (ci, [vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, i64, ci,
                                             PCFG, i64, ci, vp]),
    "tbik_tree_all_reduce_local": (ci, [C.POINTER(vp), ci, PF, i64, vp]),
    "tbik_ring_reduce_local": (ci, [C.POINTER(vp), ci, PF, i64, vp]),
    "tbik_group_create": (ci, [ci, ci, ci, i64, C.POINTER(vp)]),
    "tbik_group_ipc_handle": (ci, [vp, vp]),
    "tbik_group_open_peers": (ci, [vp, vp]),
    "tbik_group_destroy": (ci, [vp]),
    "tbik_group_send_buffer": (vp, [vp]),
    "tbik_group_world_size": (ci, [vp]),
    "tbik_group_rank": (ci, [vp]),
    "tbik_group_fused_count": (i64, [vp]),
    "tbik_tree_matmul_hostio": (ci, [vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, i64, PCFG, ci, i64, vp]),
    "tbik_group_row_parallel_forward_hostio": (ci, [vp, vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, i64, i64,
                                                    PCFG, i64, ci, i64, vp]),
    "tbik_group_tree_all_reduce": (ci, [vp, PF, PF, i64, vp]),
    "tbik_group_barrier": (ci, [vp, vp]),
    "tbik_leaf_dot": (ci, [PF, PF, i64, PF, vp]),
    "tbik_silu": (ci, [vp, ci, i64, i64, i64, PF, i64, vp]),
    "tbik_local_group_create": (ci, [ci, C.POINTER(ci), C.POINTER(vp)]),
    "tbik_local_group_destroy": (ci, [vp]),
    "tbik_local_group_device": (ci, [vp, ci]),
    "tbik_local_group_stream": (vp, [vp, ci]),
    "tbik_local_group_row_parallel_forward": (ci, [vp, C.POINTER(vp), ci, PI64, C.POINTER(vp), ci, PI64, PF, i64,
                                                   i64, i64, i64, PCFG, i64, ci, vp]),
    "tbik_baseline_gemm": (ci, [vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, i64, vp]),
    "tbik_baseline_row_parallel_forward_local": (ci, [vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, i64, ci, vp]),
    "tbik_baseline_column_parallel_forward_local": (ci, [vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, i64, ci, vp]),
    "tbik_nccl_unique_id": (ci, [vp]),
    "tbik_nccl_comm_create": (ci, [ci, ci, ci, vp, C.POINTER(vp)]),
    "tbik_nccl_comm_destroy": (ci, [vp]),
    "tbik_baseline_cublas_nccl": (ci, [vp, vp, ci, i64, vp, ci, i64, vp, i64, i64, i64, ci, vp]),
    "tbik_group_all_gather": (ci, [vp, vp, i64, i64, i64, ci, vp, i64, vp]),
    "tbik_group_logsoftmax_merge": (ci, [vp, PF, i64, PF, vp]),
    "tbik_group_row_parallel_forward": (ci, [vp, vp, ci, i64, vp, ci, i64, PF, i64, i64, i64, i64,
                                             PCFG, i64, ci, vp]),
    "tbik_tree_rmsnorm": (ci, [vp, ci, i64, PF, C.c_float, vp, ci, i64, i64, i64, vp]),
    "tbik_logsoftmax_shard_state": (ci, [PF, i64, i64, i64, i64, PF, vp]),
    "tbik_logsoftmax_shard_state_chunks": (ci, [PF, i64, i64, i64, i64, PF, vp]),
    "tbik_logsoftmax_chunk_states": (ci, [PF, i64, i64, i64, i64, PF, i64, vp]),
    "tbik_tree_matmul_logits": (ci, [vp, ci, i64, vp, ci, i64, PF, i64, PF, i64, i64, i64, i64, i64, PCFG, ci, vp]),
    "tbik_logsoftmax_merge": (ci, [C.POINTER(vp), ci, i64, PF, vp]),
    "tbik_logsoftmax_finish": (ci, [PF, i64, i64, i64, PF, PF, i64, vp, i64, PF, vp]),
    "tbik_tree_logsoftmax_local": (ci, [PF, i64, i64, i64, i64, ci, PF, PF, i64, vp, PF, vp]),
    "tbik_embedding": (ci, [vp, i64, i64, vp, i64, vp, vp]),
    "tbik_rope": (ci, [PF, i64, i64, ci, ci, vp, PF, PF, vp, i64, i64, vp]),
    "tbik_rope_qkv": (ci, [PF, i64, ci, ci, ci, vp, PF, PF, vp, vp, vp, i64, vp]),
    "tbik_cast_bf16": (ci, [PF, i64, i64, i64, vp, i64, vp]),
    "tbik_attention_prefill": (ci, [vp, i64, vp, i64, vp, i64, i64, ci, ci, ci, ci, C.c_float, vp, i64, vp]),
    "tbik_attention_prefill_tc": (ci, [vp, i64, vp, i64, vp, i64, i64, ci, ci, ci, ci, C.c_float, vp, i64, vp]),
    "tbik_silu_mul": (ci, [PF, i64, i64, i64, vp, i64, vp]),
    "tbik_residual_add": (ci, [vp, i64, PF, i64, i64, i64, vp]),
    "tbik_residual_rmsnorm": (ci, [vp, i64, PF, i64, PF, C.c_float, vp, i64, i64, i64, vp]),
    "tbik_debug_tc_stats": (ci, [C.POINTER(C.c_ulonglong), ci]),
    "tbik_matrix_write": (ci, [C.c_char_p, vp, ci, i64, i64]),
    "tbik_matrix_read_header": (ci, [C.c_char_p, C.POINTER(ci), PI64, PI64]),
    "tbik_matrix_read": (ci, [C.c_char_p, vp, i64]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

TBIK_IPC_HANDLE_BYTES = 128
TBIK_NCCL_ID_BYTES = 128


def header_functions() -> list[str]:
    """Every function the C ABI header declares (used by the export test)."""
    with open(HEADER_PATH) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tbik_[a-z0-9_]+)\s*\(", text)))
