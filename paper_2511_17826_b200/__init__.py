"""paper_2511_17826_b200 -- B200-native Tree-Based Invariant Kernels (TBIK).

The product is the sm_100a CUDA library libtbik_b200.so (csrc/) behind the C
ABI in include/tbik_b200.h; this package is its host-side mirror of the
reference C++ API (proj/include/tbik/*.hpp).  See DESIGN.md.
"""
from ._lib import ErrorCode, TbikError, header_functions, lib  # noqa: F401
from .api import (BF16, F32, LEAF_FMA, LEAF_TCGEN05, BlockConfig, DeviceGroup,  # noqa: F401
                  PeerGroup, ReductionPlan, ShardPlan, all_gather, column_parallel_forward,
                  default_block_config, device_available, launch_count, last_kernel, exchange_handles, log_softmax,
                  matrix_read, matrix_write,
                  make_column_shard_plan, make_row_shard_plan, plan_blocks, ring_reduce_baseline,
                  rmsnorm, row_parallel_forward, sync, tree_all_reduce, tree_all_reduce_per_rank,
                  tree_matmul, tree_matmul_hostio, tree_matmul_leaves, tree_matmul_silu_mul,
                  interleave_gate_up, LocalGroup, baseline_row_parallel_forward,
                  baseline_column_parallel_forward, silu, leaf_dot, set_schedule, schedule,
                  tree_matmul_logits, column_parallel_logits, chunk_states_per_row)

__version__ = "0.1.0"
