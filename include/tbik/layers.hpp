// tbik/layers.hpp -- drop-in for proj/include/tbik/layers.hpp (layers.hpp:17-56):
// column- and row-parallel TBIK linear layers over a DeviceGroup, on the B200.
// row_parallel_forward shards K by whole leaf groups (make_row_shard_plan), runs
// each rank's tree GEMM on its device with the GLOBAL k_first, and merges the
// f32 partials with the fixed-order tree all-reduce: bit-identical for every
// feasible TP size.  The baseline_* status-quo layers run cuBLAS (sequential-K
// class, order not controlled) + the left-to-right ring reduction.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "tbik/collective.hpp"
#include "tbik/matmul.hpp"
#include "tbik/matrix.hpp"

namespace tbik {

struct ShardPlan {
  enum class Mode { Column, Row };

  Mode mode;
  int tp_size;
  std::vector<std::pair<std::int64_t, std::int64_t>> bounds;
};

TBIK_CPP_API ShardPlan make_column_shard_plan(std::int64_t n, int tp_size);

TBIK_CPP_API ShardPlan make_row_shard_plan(std::int64_t k, const BlockConfig& cfg, int tp_size, std::int64_t c_max);

TBIK_CPP_API Matrix column_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group,
                                            const BlockConfig& cfg);

TBIK_CPP_API Matrix row_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group,
                                         const BlockConfig& cfg, std::int64_t c_max = 8);

TBIK_CPP_API Matrix baseline_row_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group);

TBIK_CPP_API Matrix baseline_column_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group);

// ---- B200 additions: explicit leaf ----
TBIK_CPP_API Matrix column_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group,
                                            const BlockConfig& cfg, Leaf leaf);
TBIK_CPP_API Matrix row_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group,
                                         const BlockConfig& cfg, std::int64_t c_max, Leaf leaf);

}  // namespace tbik
