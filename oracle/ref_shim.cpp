// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libtbik_ref.so).  It lets the pytest suite and bench.py's
// reference arm call the reference's own C++ API with plain pointers:
//
//   ref_tree_matmul            -> tbik::tree_matmul            (matmul.hpp:53)
//   ref_row_parallel_forward   -> tbik::row_parallel_forward   (layers.hpp:43-45)
//   ref_column_parallel_forward-> tbik::column_parallel_forward(layers.hpp:36-38)
//   ref_global_tree_matmul     -> tbik::oracle::global_tree_matmul (oracle.hpp:46-47)
//   ref_tree_all_reduce        -> tbik::tree_all_reduce        (collective.hpp:38-39)
//   ...
//
// Error convention: 0 = ok, 1 + int(tbik::ErrorCode) for a TbikError
// (errors.hpp:8-20), 100 for any other exception.  This is the same mapping
// the product's C ABI uses (include/tbik_b200.h), so error parity can be
// checked code-for-code.

#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "tbik/collective.hpp"
#include "tbik/demo.hpp"
#include "tbik/errors.hpp"
#include "tbik/layers.hpp"
#include "tbik/matmul.hpp"
#include "tbik/matrix.hpp"
#include "tbik/oracle.hpp"
#include "tbik/runner.hpp"
#include "tbik/threading.hpp"
#include "tbik/witness.hpp"

using namespace tbik;

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const TbikError& e) {
    return 1 + static_cast<int>(e.code());
  } catch (...) {
    return 100;
  }
}

// dtype: 0 = f32, 1 = bf16 (matrix.hpp:20)
Matrix make_matrix(const void* p, int dtype, std::int64_t rows,
                   std::int64_t cols) {
  const std::size_t n = static_cast<std::size_t>(rows * cols);
  if (dtype == 0) {
    std::vector<float> v(n);
    std::memcpy(v.data(), p, n * sizeof(float));
    return Matrix::from_f32(rows, cols, std::move(v));
  }
  std::vector<std::uint16_t> v(n);
  std::memcpy(v.data(), p, n * sizeof(std::uint16_t));
  return Matrix::from_bf16(rows, cols, std::move(v));
}

void store_f32(const Matrix& m, float* out) {
  const auto& d = m.f32_data();
  std::memcpy(out, d.data(), d.size() * sizeof(float));
}

BlockConfig make_cfg(const std::int64_t cfg[4]) {
  return BlockConfig{cfg[0], cfg[1], cfg[2], cfg[3]};
}

}  // namespace

extern "C" {

void ref_set_threads(int n) { set_worker_count(n); }
int ref_worker_count() { return worker_count(); }

int ref_plan_blocks(std::int64_t K, const std::int64_t cfg[4],
                    std::int64_t c_max, std::int64_t out[4]) {
  return guarded([&] {
    ReductionPlan p = plan_blocks(K, make_cfg(cfg), c_max);
    out[0] = p.tiles_total;
    out[1] = p.k_first;
    out[2] = p.leaves;
    out[3] = p.depth;
  });
}

int ref_make_row_shard_plan(std::int64_t K, const std::int64_t cfg[4], int tp,
                            std::int64_t c_max, std::int64_t* bounds) {
  return guarded([&] {
    ShardPlan s = make_row_shard_plan(K, make_cfg(cfg), tp, c_max);
    for (int r = 0; r < tp; ++r) {
      bounds[2 * r] = s.bounds[static_cast<std::size_t>(r)].first;
      bounds[2 * r + 1] = s.bounds[static_cast<std::size_t>(r)].second;
    }
  });
}

int ref_make_column_shard_plan(std::int64_t N, int tp, std::int64_t* bounds) {
  return guarded([&] {
    ShardPlan s = make_column_shard_plan(N, tp);
    for (int r = 0; r < tp; ++r) {
      bounds[2 * r] = s.bounds[static_cast<std::size_t>(r)].first;
      bounds[2 * r + 1] = s.bounds[static_cast<std::size_t>(r)].second;
    }
  });
}

int ref_random_normal(std::uint64_t seed, std::uint64_t stream,
                      std::int64_t rows, std::int64_t cols, int dtype,
                      float mean, float stddev, void* out) {
  return guarded([&] {
    Rng rng(seed, stream);
    Matrix m = matrix_random_normal(rng, rows, cols,
                                    dtype == 0 ? Dtype::F32 : Dtype::Bf16, mean,
                                    stddev);
    if (dtype == 0) {
      std::memcpy(out, m.f32_data().data(), m.f32_data().size() * 4);
    } else {
      std::memcpy(out, m.bf16_data().data(), m.bf16_data().size() * 2);
    }
  });
}

std::uint64_t ref_fingerprint(const void* p, int dtype, std::int64_t rows,
                              std::int64_t cols) {
  return bit_fingerprint(make_matrix(p, dtype, rows, cols));
}

std::uint16_t ref_bf16_round(float x) { return bf16_round(x).bits; }

float ref_leaf_dot(const float* a, const float* b, std::int64_t n) {
  return leaf_dot(a, b, n);
}

int ref_tree_reduce(const float* leaves, std::int64_t n, float* out) {
  return guarded([&] {
    *out = oracle::tree_reduce(std::span<const float>(leaves, static_cast<std::size_t>(n)));
  });
}

int ref_tree_matmul(const void* a, int adt, const void* b, int bdt,
                    std::int64_t M, std::int64_t K, std::int64_t N,
                    const std::int64_t cfg[4], float* out) {
  return guarded([&] {
    store_f32(tree_matmul(make_matrix(a, adt, M, K), make_matrix(b, bdt, K, N),
                          make_cfg(cfg)),
              out);
  });
}

int ref_row_parallel_forward(const void* a, int adt, const void* b, int bdt,
                             std::int64_t M, std::int64_t K, std::int64_t N,
                             const std::int64_t cfg[4], int tp,
                             std::int64_t c_max, float* out) {
  return guarded([&] {
    DeviceGroup g(tp);
    store_f32(row_parallel_forward(make_matrix(a, adt, M, K),
                                   make_matrix(b, bdt, K, N), g, make_cfg(cfg),
                                   c_max),
              out);
  });
}

int ref_column_parallel_forward(const void* a, int adt, const void* b, int bdt,
                                std::int64_t M, std::int64_t K, std::int64_t N,
                                const std::int64_t cfg[4], int tp, float* out) {
  return guarded([&] {
    DeviceGroup g(tp);
    store_f32(column_parallel_forward(make_matrix(a, adt, M, K),
                                      make_matrix(b, bdt, K, N), g,
                                      make_cfg(cfg)),
              out);
  });
}

int ref_baseline_row_parallel_forward(const void* a, int adt, const void* b,
                                      int bdt, std::int64_t M, std::int64_t K,
                                      std::int64_t N, int tp, float* out) {
  return guarded([&] {
    DeviceGroup g(tp);
    store_f32(baseline_row_parallel_forward(make_matrix(a, adt, M, K),
                                            make_matrix(b, bdt, K, N), g),
              out);
  });
}

int ref_global_tree_matmul(const void* a, int adt, const void* b, int bdt,
                           std::int64_t M, std::int64_t K, std::int64_t N,
                           const std::int64_t cfg[4], std::int64_t c_max,
                           float* out) {
  return guarded([&] {
    store_f32(oracle::global_tree_matmul(make_matrix(a, adt, M, K),
                                         make_matrix(b, bdt, K, N),
                                         make_cfg(cfg), c_max),
              out);
  });
}

int ref_sequential_matmul(const void* a, int adt, const void* b, int bdt,
                          std::int64_t M, std::int64_t K, std::int64_t N,
                          float* out) {
  return guarded([&] {
    store_f32(oracle::sequential_matmul_f32(make_matrix(a, adt, M, K),
                                            make_matrix(b, bdt, K, N)),
              out);
  });
}

// contributions: W consecutive blocks of rows*cols f32.
int ref_tree_all_reduce(const float* contributions, int W, std::int64_t rows,
                        std::int64_t cols, float* out) {
  return guarded([&] {
    DeviceGroup g(W);
    std::vector<Matrix> xs;
    for (int r = 0; r < W; ++r) {
      xs.push_back(make_matrix(contributions + r * rows * cols, 0, rows, cols));
    }
    store_f32(tree_all_reduce(g, xs), out);
  });
}

int ref_ring_reduce(const float* contributions, int W, std::int64_t rows,
                    std::int64_t cols, float* out) {
  return guarded([&] {
    DeviceGroup g(W);
    std::vector<Matrix> xs;
    for (int r = 0; r < W; ++r) {
      xs.push_back(make_matrix(contributions + r * rows * cols, 0, rows, cols));
    }
    store_f32(ring_reduce_baseline(g, xs), out);
  });
}

int ref_device_group(int W) {
  return guarded([&] { DeviceGroup g(W); });
}

int ref_rmsnorm(const void* x, int dt, std::int64_t rows, std::int64_t cols,
                const float* gamma, float eps, float* out) {
  return guarded([&] {
    std::vector<float> g(gamma, gamma + cols);
    store_f32(rmsnorm(make_matrix(x, dt, rows, cols), g, eps), out);
  });
}

int ref_silu(const void* x, int dt, std::int64_t rows, std::int64_t cols,
             float* out) {
  return guarded([&] { store_f32(silu(make_matrix(x, dt, rows, cols)), out); });
}

// The reference's own acceptance checks (runner.hpp:50-77); pass -> 1.
int ref_check_theorem1_exhaustive(int max_t, int vectors,
                                  std::uint64_t* failures) {
  CheckResult r = check_theorem1_exhaustive(max_t, vectors);
  *failures = r.bit_diff_count;
  return r.pass ? 1 : 0;
}

int ref_check_collective_symmetry(int vectors, std::int64_t elems,
                                  std::uint64_t* diffs) {
  CheckResult r = check_collective_symmetry({1, 2, 4, 8}, vectors, elems);
  *diffs = r.bit_diff_count;
  return r.pass ? 1 : 0;
}

int ref_check_kernel_tp_invariance(int seeds, std::int64_t m, std::int64_t k,
                                   std::int64_t n, std::uint64_t* diffs) {
  CheckResult r = check_kernel_tp_invariance(
      Dtype::Bf16, default_block_config(Dtype::Bf16), {1, 2, 4, 8}, seeds, m, k,
      n);
  *diffs = r.bit_diff_count;
  return r.pass ? 1 : 0;
}

// Witnesses (witness.hpp) used as known-answer tests.
void ref_nonassoc_witness(float out[7]) {
  NonassocWitness w = find_nonassoc_witness();
  out[0] = w.a;
  out[1] = w.b;
  out[2] = w.c;
  out[3] = w.left_first;
  out[4] = w.right_first;
  out[5] = w.sequential;
  out[6] = w.tree;
}

void ref_fma_witness(float out[5]) {
  FmaWitness w = find_fma_witness();
  out[0] = w.a;
  out[1] = w.b;
  out[2] = w.c;
  out[3] = w.fused;
  out[4] = w.two_step;
}

std::uint64_t ref_leaf_order_witness(float a[8], float b[8], float out[2]) {
  LeafOrderWitness w = find_leaf_order_witness();
  std::memcpy(a, w.a.data(), 8 * sizeof(float));
  std::memcpy(b, w.b.data(), 8 * sizeof(float));
  out[0] = w.ascending;
  out[1] = w.descending;
  return w.seed;
}

// matrix_write / matrix_read (matrix.hpp:86-87), unmodified reference code.
int ref_matrix_write(const char* path, const void* data, int dtype, std::int64_t rows, std::int64_t cols) {
  return guarded([&] { matrix_write(path, make_matrix(data, dtype, rows, cols)); });
}

// Reads a TBIK file with the reference; fills dims/dtype and copies the
// payload when `out` is non-null (capacity in bytes).
int ref_matrix_read(const char* path, int* dtype, std::int64_t* rows, std::int64_t* cols, void* out,
                    std::int64_t capacity) {
  return guarded([&] {
    Matrix m = matrix_read(path);
    *dtype = static_cast<int>(m.dtype());
    *rows = m.rows();
    *cols = m.cols();
    if (!out) return;
    if (m.dtype() == Dtype::F32) {
      const auto& d = m.f32_data();
      if (static_cast<std::int64_t>(d.size() * 4) <= capacity) std::memcpy(out, d.data(), d.size() * 4);
    } else {
      const auto& d = m.bf16_data();
      if (static_cast<std::int64_t>(d.size() * 2) <= capacity) std::memcpy(out, d.data(), d.size() * 2);
    }
  });
}

}  // extern "C"
