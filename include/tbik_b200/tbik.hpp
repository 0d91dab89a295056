// tbik_b200/tbik.hpp -- drop-in C++ mirror of the reference API
// (/root/reference/proj/include/tbik/{errors,matrix,rng,matmul,collective,layers,demo}.hpp)
// implemented on the B200 through the C ABI (include/tbik_b200.h).
//
// Same names, argument meaning, value semantics and error behaviour as the
// reference: Matrix owns host storage and is returned by value; failures throw
// tbik::TbikError carrying the reference's ErrorCode.  Every compute call
// uploads its operands, runs the sm_100a kernels and downloads the result
// (use the C ABI directly to keep data resident on the GPU).  There is no CPU
// fallback: without an sm_100 device the calls throw (status NoDevice).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tbik_b200.h"

#if defined(__GNUC__)
#define TBIK_CPP_API __attribute__((visibility("default")))
#else
#define TBIK_CPP_API
#endif

namespace tbik {

// ---- errors.hpp:8-35 ----------------------------------------------------------
enum class ErrorCode {
  BadDimension,
  ShapeMismatch,
  BadMagic,
  Truncated,
  UnknownDtype,
  PlanInfeasible,
  ShardError,
  BadWorldSize,
  CollectiveMismatch,
  BadArgument,
  Io,
};

class TbikError : public std::runtime_error {
 public:
  TbikError(ErrorCode code, const std::string& what, int status = 0)
      : std::runtime_error(what), code_(code), status_(status) {}
  ErrorCode code() const { return code_; }
  // The raw tbik_status (>= 100 for device conditions: CudaError, NoDevice, Unsupported).
  int status() const { return status_; }

 private:
  ErrorCode code_;
  int status_;
};

[[noreturn]] TBIK_CPP_API void fail(ErrorCode code, const std::string& what);
// Throws TbikError for a non-zero tbik_status (device codes map to BadArgument
// with status() telling them apart).
TBIK_CPP_API void check_status(int status);

// ---- numerics.hpp:21-62 ---------------------------------------------------------
inline std::uint32_t f32_bits(float x) {
  std::uint32_t u;
  std::memcpy(&u, &x, 4);
  return u;
}
inline float f32_from_bits(std::uint32_t u) {
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}
struct Bf16 {
  std::uint16_t bits = 0;
  friend bool operator==(Bf16 a, Bf16 b) { return a.bits == b.bits; }
};
inline constexpr std::uint16_t kBf16CanonicalNan = 0x7FC0;
inline float bf16_to_f32(Bf16 v) { return f32_from_bits(static_cast<std::uint32_t>(v.bits) << 16); }
inline Bf16 bf16_round(float x) {
  std::uint32_t u = f32_bits(x);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu) != 0) return Bf16{kBf16CanonicalNan};
  return Bf16{static_cast<std::uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16)};
}
inline bool f32_bit_equal(float a, float b) { return f32_bits(a) == f32_bits(b); }

// ---- rng.hpp:15-60 (counter-based SplitMix64 + Box-Muller) ----------------------
class Rng {
 public:
  explicit Rng(std::uint64_t seed, std::uint64_t stream = 0) : seed_(seed), stream_(stream) {}
  std::uint64_t next_u64() { return mix64(counter_++ ^ mix64(stream_ ^ mix64(seed_ + 0x9E3779B97F4A7C15ull))); }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u1 = 1.0 - next_unit();
    double u2 = next_unit();
    double r = std::sqrt(-2.0 * std::log(u1));
    double theta = 2.0 * 3.14159265358979323846 * u2;
    spare_ = r * std::sin(theta);
    has_spare_ = true;
    return r * std::cos(theta);
  }
  static std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }

 private:
  std::uint64_t seed_, stream_, counter_ = 0;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

// ---- matrix.hpp:18-89 -------------------------------------------------------------
enum class Dtype : std::uint16_t { F32 = 0, Bf16 = 1 };
TBIK_CPP_API const char* dtype_name(Dtype d);

class TBIK_CPP_API Matrix {
 public:
  Matrix() = default;
  Matrix(std::int64_t rows, std::int64_t cols, Dtype dtype);
  static Matrix from_f32(std::int64_t rows, std::int64_t cols, std::vector<float> data);
  static Matrix from_bf16(std::int64_t rows, std::int64_t cols, std::vector<std::uint16_t> data);

  std::int64_t rows() const { return rows_; }
  std::int64_t cols() const { return cols_; }
  std::int64_t size() const { return rows_ * cols_; }
  Dtype dtype() const { return dtype_; }
  float at(std::int64_t r, std::int64_t c) const {
    const std::int64_t i = r * cols_ + c;
    return dtype_ == Dtype::F32 ? f32_[i] : bf16_to_f32(Bf16{bf16_[i]});
  }
  void set(std::int64_t r, std::int64_t c, float v) {
    const std::int64_t i = r * cols_ + c;
    if (dtype_ == Dtype::F32)
      f32_[i] = v;
    else
      bf16_[i] = bf16_round(v).bits;
  }
  const std::vector<float>& f32_data() const;
  std::vector<float>& f32_data();
  const std::vector<std::uint16_t>& bf16_data() const;
  std::vector<float> widened() const;
  Matrix slice_cols(std::int64_t begin, std::int64_t end) const;
  Matrix slice_rows(std::int64_t begin, std::int64_t end) const;
  const void* raw() const { return dtype_ == Dtype::F32 ? static_cast<const void*>(f32_.data()) : bf16_.data(); }
  std::size_t raw_bytes() const { return static_cast<std::size_t>(size()) * (dtype_ == Dtype::F32 ? 4 : 2); }

 private:
  std::int64_t rows_ = 0, cols_ = 0;
  Dtype dtype_ = Dtype::F32;
  std::vector<float> f32_;
  std::vector<std::uint16_t> bf16_;
};

TBIK_CPP_API Matrix cast_to_bf16(const Matrix& m);
TBIK_CPP_API Matrix cast_to_f32(const Matrix& m);
TBIK_CPP_API bool bit_equal(const Matrix& a, const Matrix& b);
TBIK_CPP_API std::uint64_t bit_diff_count(const Matrix& a, const Matrix& b);
TBIK_CPP_API std::uint64_t bit_fingerprint(const Matrix& m);
TBIK_CPP_API Matrix matrix_random_normal(Rng& rng, std::int64_t rows, std::int64_t cols, Dtype dtype,
                                         float mean, float stddev);
// matrix.hpp:86-87: the TBIK file format (tbik_matrix_write / tbik_matrix_read).
TBIK_CPP_API void matrix_write(const std::string& path, const Matrix& m);
TBIK_CPP_API Matrix matrix_read(const std::string& path);

// ---- matmul.hpp:18-53 ----------------------------------------------------------
struct BlockConfig {
  std::int64_t block_m = 0;
  std::int64_t block_k = 0;
  std::int64_t block_n = 0;
  std::int64_t k_first = 0;
};
struct ReductionPlan {
  std::int64_t tiles_total = 0;
  std::int64_t k_first = 1;
  std::int64_t leaves = 0;
  std::int64_t depth = 0;
};
// B200 extension: which computation forms a leaf (see tbik_leaf_mode).
enum class Leaf { Fma = TBIK_LEAF_FMA, Tcgen05 = TBIK_LEAF_TCGEN05 };

TBIK_CPP_API BlockConfig default_block_config(Dtype dtype);
TBIK_CPP_API bool is_power_of_two(std::int64_t v);
TBIK_CPP_API ReductionPlan plan_blocks(std::int64_t K, const BlockConfig& cfg, std::int64_t c_max);
TBIK_CPP_API Matrix tree_matmul(const Matrix& a, const Matrix& b, const BlockConfig& cfg,
                                Leaf leaf = Leaf::Tcgen05);

// ---- collective.hpp:15-45 --------------------------------------------------------
class TBIK_CPP_API DeviceGroup {
 public:
  explicit DeviceGroup(int world_size);
  int world_size() const { return world_size_; }

 private:
  int world_size_;
};
TBIK_CPP_API std::vector<Matrix> all_gather(const DeviceGroup& group, const std::vector<Matrix>& x_per_rank);
TBIK_CPP_API std::vector<Matrix> tree_all_reduce_per_rank(const DeviceGroup& group,
                                                          const std::vector<Matrix>& x_per_rank);
TBIK_CPP_API Matrix tree_all_reduce(const DeviceGroup& group, const std::vector<Matrix>& x_per_rank);
TBIK_CPP_API Matrix ring_reduce_baseline(const DeviceGroup& group, const std::vector<Matrix>& x_per_rank);

// ---- layers.hpp:17-56 --------------------------------------------------------------
struct ShardPlan {
  enum class Mode { Column, Row };
  Mode mode;
  int tp_size;
  std::vector<std::pair<std::int64_t, std::int64_t>> bounds;
};
TBIK_CPP_API ShardPlan make_column_shard_plan(std::int64_t n, int tp_size);
TBIK_CPP_API ShardPlan make_row_shard_plan(std::int64_t k, const BlockConfig& cfg, int tp_size, std::int64_t c_max);
TBIK_CPP_API Matrix column_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group,
                                            const BlockConfig& cfg, Leaf leaf = Leaf::Tcgen05);
TBIK_CPP_API Matrix row_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group,
                                         const BlockConfig& cfg, std::int64_t c_max = 8,
                                         Leaf leaf = Leaf::Tcgen05);

// ---- demo.hpp:53 (tree-ordered on the GPU) ----------------------
TBIK_CPP_API Matrix rmsnorm(const Matrix& x, const std::vector<float>& gamma, float eps);

}  // namespace tbik
