// tbik/matmul.hpp -- drop-in for proj/include/tbik/matmul.hpp (matmul.hpp:18-55):
// the TP-invariant tree GEMM.  Same declarations; tree_matmul runs on the B200
// (sm_100a kernels through the C ABI, include/tbik_b200.h).
//
// The leaf (one block_k tile dot product, matmul.cpp:69-75) is selectable --
// a B200 addition:
//   Leaf::Fma      CUDA-core ascending-k fma chain from +0: bit-identical to the
//                  reference for every input (the default, so an unmodified
//                  caller gets the reference's bits);
//   Leaf::Tcgen05  tcgen05.mma leaves (bf16 only, block_k % 64 == 0; throws
//                  Unsupported otherwise): every merge above the leaf is still
//                  the reference's f32 tree; the leaf is ulp-bounded
//                  (DESIGN.md section 3).  TP- and batch-invariant like Fma.
// set_default_leaf() switches the leaf of the reference-signature calls
// process-wide; the overloads taking a Leaf pick it per call.
#pragma once

#include <cstdint>

#include "tbik/matrix.hpp"

namespace tbik {

struct BlockConfig {
  std::int64_t block_m = 0;
  std::int64_t block_k = 0;
  std::int64_t block_n = 0;
  std::int64_t k_first = 0;  // 0 = smallest feasible (plan_blocks)
};

TBIK_CPP_API BlockConfig default_block_config(Dtype dtype);

struct ReductionPlan {
  std::int64_t tiles_total = 0;
  std::int64_t k_first = 1;
  std::int64_t leaves = 0;
  std::int64_t depth = 0;
};

TBIK_CPP_API bool is_power_of_two(std::int64_t v);
TBIK_CPP_API std::int64_t log2_exact(std::int64_t v);

TBIK_CPP_API ReductionPlan plan_blocks(std::int64_t K, const BlockConfig& cfg, std::int64_t c_max);

// Leaf semantics (ascending-k fma from +0), evaluated by one GPU thread.
TBIK_CPP_API float leaf_dot(const float* a, const float* b, std::int64_t n);

TBIK_CPP_API Matrix tree_matmul(const Matrix& a, const Matrix& b, const BlockConfig& cfg);

// ---- B200 additions ----
enum class Leaf { Fma = 0, Tcgen05 = 1 };  // = tbik_leaf_mode
TBIK_CPP_API void set_default_leaf(Leaf leaf);
TBIK_CPP_API Leaf default_leaf();
TBIK_CPP_API Matrix tree_matmul(const Matrix& a, const Matrix& b, const BlockConfig& cfg, Leaf leaf);

}  // namespace tbik
