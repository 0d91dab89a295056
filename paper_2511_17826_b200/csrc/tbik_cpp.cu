// tbik_cpp.cu -- host implementation of the drop-in C++ API (include/tbik/*.hpp,
// the reference's proj/include/tbik/ declarations).
//
// Matrix / Rng / fingerprint semantics restate the reference's
// (matrix.cpp:11-181); every compute entry uploads operands to the device(s)
// of the DeviceGroup, calls the C ABI (tbik_b200.h) and downloads the result.
// Errors come back as tbik::TbikError with the reference's ErrorCode.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "tbik_b200.h"
#include "tbik_b200/tbik.hpp"

namespace tbik {

void fail(ErrorCode code, const std::string& what) { throw TbikError(code, what); }

void check_status(int st) {
  if (st == TBIK_OK) return;
  const std::string what = std::string(tbik_status_string(st)) + ": " + tbik_last_error();
  if (st >= 1 && st <= 11) throw TbikError(static_cast<ErrorCode>(st - 1), what, st);
  throw TbikError(ErrorCode::BadArgument, what, st);
}

const char* dtype_name(Dtype d) { return d == Dtype::F32 ? "f32" : "bf16"; }

// ---- Matrix (matrix.cpp:13-100) ------------------------------------------------
Matrix::Matrix(std::int64_t rows, std::int64_t cols, Dtype dtype) : rows_(rows), cols_(cols), dtype_(dtype) {
  if (rows < 1 || cols < 1)
    fail(ErrorCode::BadDimension,
         "matrix dimensions must be >= 1, got " + std::to_string(rows) + "x" + std::to_string(cols));
  if (dtype_ == Dtype::F32)
    f32_.assign(static_cast<std::size_t>(rows * cols), 0.0f);
  else
    bf16_.assign(static_cast<std::size_t>(rows * cols), 0);
}

Matrix Matrix::from_f32(std::int64_t rows, std::int64_t cols, std::vector<float> data) {
  Matrix m(rows, cols, Dtype::F32);
  if (static_cast<std::int64_t>(data.size()) != rows * cols)
    fail(ErrorCode::BadDimension, "payload length does not match dimensions");
  m.f32_ = std::move(data);
  return m;
}

Matrix Matrix::from_bf16(std::int64_t rows, std::int64_t cols, std::vector<std::uint16_t> data) {
  Matrix m(rows, cols, Dtype::Bf16);
  if (static_cast<std::int64_t>(data.size()) != rows * cols)
    fail(ErrorCode::BadDimension, "payload length does not match dimensions");
  m.bf16_ = std::move(data);
  return m;
}

const std::vector<float>& Matrix::f32_data() const {
  if (dtype_ != Dtype::F32) fail(ErrorCode::BadArgument, "matrix is not f32");
  return f32_;
}
std::vector<float>& Matrix::f32_data() {
  if (dtype_ != Dtype::F32) fail(ErrorCode::BadArgument, "matrix is not f32");
  return f32_;
}
const std::vector<std::uint16_t>& Matrix::bf16_data() const {
  if (dtype_ != Dtype::Bf16) fail(ErrorCode::BadArgument, "matrix is not bf16");
  return bf16_;
}

std::vector<float> Matrix::widened() const {
  if (dtype_ == Dtype::F32) return f32_;
  std::vector<float> out(bf16_.size());
  for (std::size_t i = 0; i < bf16_.size(); ++i) out[i] = bf16_to_f32(Bf16{bf16_[i]});
  return out;
}

Matrix Matrix::slice_cols(std::int64_t b, std::int64_t e) const {
  if (b < 0 || e > cols_ || b >= e) fail(ErrorCode::BadDimension, "bad column slice");
  Matrix out(rows_, e - b, dtype_);
  const std::size_t es = dtype_ == Dtype::F32 ? 4 : 2;
  for (std::int64_t r = 0; r < rows_; ++r)
    std::memcpy(static_cast<char*>(const_cast<void*>(out.raw())) + r * (e - b) * es,
                static_cast<const char*>(raw()) + (r * cols_ + b) * es, static_cast<std::size_t>(e - b) * es);
  return out;
}

Matrix Matrix::slice_rows(std::int64_t b, std::int64_t e) const {
  if (b < 0 || e > rows_ || b >= e) fail(ErrorCode::BadDimension, "bad row slice");
  Matrix out(e - b, cols_, dtype_);
  const std::size_t es = dtype_ == Dtype::F32 ? 4 : 2;
  std::memcpy(const_cast<void*>(out.raw()), static_cast<const char*>(raw()) + b * cols_ * es, out.raw_bytes());
  return out;
}

Matrix cast_to_bf16(const Matrix& m) {
  if (m.dtype() == Dtype::Bf16) return m;
  std::vector<std::uint16_t> d(static_cast<std::size_t>(m.size()));
  const auto& s = m.f32_data();
  for (std::size_t i = 0; i < d.size(); ++i) d[i] = bf16_round(s[i]).bits;
  return Matrix::from_bf16(m.rows(), m.cols(), std::move(d));
}

Matrix cast_to_f32(const Matrix& m) {
  if (m.dtype() == Dtype::F32) return m;
  return Matrix::from_f32(m.rows(), m.cols(), m.widened());
}

std::uint64_t bit_diff_count(const Matrix& a, const Matrix& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols() || a.dtype() != b.dtype()) return ~std::uint64_t{0};
  std::uint64_t d = 0;
  if (a.dtype() == Dtype::F32) {
    for (std::size_t i = 0; i < a.f32_data().size(); ++i) d += f32_bits(a.f32_data()[i]) != f32_bits(b.f32_data()[i]);
  } else {
    for (std::size_t i = 0; i < a.bf16_data().size(); ++i) d += a.bf16_data()[i] != b.bf16_data()[i];
  }
  return d;
}

bool bit_equal(const Matrix& a, const Matrix& b) { return bit_diff_count(a, b) == 0; }

std::uint64_t bit_fingerprint(const Matrix& m) {  // FNV-1a, matrix.cpp:143-161
  std::uint64_t h = 0xCBF29CE484222325ull;
  auto feed = [&h](const void* p, std::size_t n) {
    const auto* c = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) {
      h ^= c[i];
      h *= 0x100000001B3ull;
    }
  };
  std::uint64_t dims[2] = {static_cast<std::uint64_t>(m.rows()), static_cast<std::uint64_t>(m.cols())};
  feed(dims, sizeof(dims));
  feed(m.raw(), m.raw_bytes());
  return h;
}

Matrix matrix_random_normal(Rng& rng, std::int64_t rows, std::int64_t cols, Dtype dtype, float mean, float stddev) {
  if (rows < 1 || cols < 1) fail(ErrorCode::BadDimension, "matrix_random_normal requires rows, cols >= 1");
  if (stddev < 0.0f) fail(ErrorCode::BadArgument, "matrix_random_normal requires stddev >= 0");
  Matrix m(rows, cols, dtype);
  for (std::int64_t r = 0; r < rows; ++r)
    for (std::int64_t c = 0; c < cols; ++c) {
      const double z = rng.next_normal();
      m.set(r, c, static_cast<float>(static_cast<double>(mean) + static_cast<double>(stddev) * z));
    }
  return m;
}

// ---- device plumbing -------------------------------------------------------------
namespace {

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(std::size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) throw TbikError(ErrorCode::BadArgument, std::string("cudaMalloc: ") + cudaGetErrorString(e), TBIK_CUDA_ERROR);
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw TbikError(ErrorCode::BadArgument, std::string(what) + ": " + cudaGetErrorString(e), TBIK_CUDA_ERROR);
}

DevBuf upload(const Matrix& m) {
  DevBuf d(m.raw_bytes());
  cuda_ok(cudaMemcpy(d.p, m.raw(), m.raw_bytes(), cudaMemcpyHostToDevice), "upload");
  return d;
}

Matrix download_f32(const DevBuf& d, std::int64_t rows, std::int64_t cols) {
  std::vector<float> v(static_cast<std::size_t>(rows * cols));
  cuda_ok(cudaMemcpy(v.data(), d.p, v.size() * 4, cudaMemcpyDeviceToHost), "download");
  return Matrix::from_f32(rows, cols, std::move(v));
}

tbik_block_config c_cfg(const BlockConfig& c) { return tbik_block_config{c.block_m, c.block_k, c.block_n, c.k_first}; }

void require_uniform(const DeviceGroup& g, const std::vector<Matrix>& xs) {  // collective.cpp:20-36
  if (static_cast<int>(xs.size()) != g.world_size())
    fail(ErrorCode::CollectiveMismatch,
         "expected " + std::to_string(g.world_size()) + " contributions, got " + std::to_string(xs.size()));
  for (std::size_t r = 1; r < xs.size(); ++r)
    if (xs[r].rows() != xs[0].rows() || xs[r].cols() != xs[0].cols() || xs[r].dtype() != xs[0].dtype())
      fail(ErrorCode::CollectiveMismatch, "rank " + std::to_string(r) + " contribution shape/dtype differs");
}

Matrix reduce(const DeviceGroup& g, const std::vector<Matrix>& xs, bool ring) {
  require_uniform(g, xs);
  if (xs[0].dtype() != Dtype::F32)
    fail(ErrorCode::CollectiveMismatch, ring ? "ring_reduce expects f32 inputs" : "tree_all_reduce expects f32 inputs");
  std::vector<DevBuf*> bufs;
  std::vector<const float*> ptrs;
  std::vector<std::unique_ptr<DevBuf>> own;
  for (const Matrix& m : xs) {
    own.emplace_back(new DevBuf(m.raw_bytes()));
    cuda_ok(cudaMemcpy(own.back()->p, m.raw(), m.raw_bytes(), cudaMemcpyHostToDevice), "upload");
    ptrs.push_back(static_cast<const float*>(own.back()->p));
  }
  DevBuf out(xs[0].raw_bytes());
  const int W = g.world_size();
  check_status(ring ? tbik_ring_reduce_local(ptrs.data(), W, static_cast<float*>(out.p), xs[0].size(), nullptr)
                    : tbik_tree_all_reduce_local(ptrs.data(), W, static_cast<float*>(out.p), xs[0].size(), nullptr));
  check_status(tbik_sync(nullptr));
  return download_f32(out, xs[0].rows(), xs[0].cols());
}

}  // namespace

// ---- matmul.hpp ----------------------------------------------------------------------
BlockConfig default_block_config(Dtype dtype) {
  tbik_block_config c;
  check_status(tbik_default_block_config(static_cast<int>(dtype), &c));
  return BlockConfig{c.block_m, c.block_k, c.block_n, c.k_first};
}

bool is_power_of_two(std::int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

std::int64_t log2_exact(std::int64_t v) {  // matmul.cpp:18-22
  std::int64_t l = 0;
  while ((std::int64_t{1} << l) < v) ++l;
  return l;
}

namespace {
std::atomic<int> g_default_leaf{static_cast<int>(Leaf::Fma)};  // the reference's bits unless asked otherwise
}
void set_default_leaf(Leaf leaf) { g_default_leaf.store(static_cast<int>(leaf)); }
Leaf default_leaf() { return static_cast<Leaf>(g_default_leaf.load()); }

float leaf_dot(const float* a, const float* b, std::int64_t n) {
  if (n < 0) fail(ErrorCode::BadDimension, "leaf_dot: n must be >= 0");
  const std::size_t bytes = static_cast<std::size_t>(n) * 4;
  DevBuf da(bytes), db(bytes), dout(4);
  if (n > 0) {
    cuda_ok(cudaMemcpy(da.p, a, bytes, cudaMemcpyHostToDevice), "upload");
    cuda_ok(cudaMemcpy(db.p, b, bytes, cudaMemcpyHostToDevice), "upload");
  }
  check_status(tbik_leaf_dot(static_cast<const float*>(da.p), static_cast<const float*>(db.p), n,
                             static_cast<float*>(dout.p), nullptr));
  check_status(tbik_sync(nullptr));
  float r = 0.0f;
  cuda_ok(cudaMemcpy(&r, dout.p, 4, cudaMemcpyDeviceToHost), "download");
  return r;
}

ReductionPlan plan_blocks(std::int64_t K, const BlockConfig& cfg, std::int64_t c_max) {
  tbik_block_config c = c_cfg(cfg);
  tbik_reduction_plan p;
  check_status(tbik_plan_blocks(K, &c, c_max, &p));
  return ReductionPlan{p.tiles_total, p.k_first, p.leaves, p.depth};
}

Matrix tree_matmul(const Matrix& a, const Matrix& b, const BlockConfig& cfg) {
  return tree_matmul(a, b, cfg, default_leaf());
}

Matrix tree_matmul(const Matrix& a, const Matrix& b, const BlockConfig& cfg, Leaf leaf) {
  if (a.cols() != b.rows())
    fail(ErrorCode::ShapeMismatch,
         "tree_matmul: inner dimensions differ, " + std::to_string(a.cols()) + " vs " + std::to_string(b.rows()));
  // The weights go to the device once; the activations stream host -> device and
  // the f32 result device -> host in row chunks overlapped with the GEMM
  // (tbik_tree_matmul_hostio) -- the reference's Matrix-in / Matrix-out call.
  DevBuf db = upload(b);
  std::vector<float> out(static_cast<std::size_t>(a.rows() * b.cols()));
  tbik_block_config c = c_cfg(cfg);
  check_status(tbik_tree_matmul_hostio(a.raw(), static_cast<int>(a.dtype()), a.cols(), db.p,
                                       static_cast<int>(b.dtype()), b.cols(), out.data(), b.cols(), a.rows(),
                                       b.cols(), a.cols(), &c, static_cast<int>(leaf), 0, nullptr));
  check_status(tbik_sync(nullptr));
  return Matrix::from_f32(a.rows(), b.cols(), std::move(out));
}

// ---- collective.hpp --------------------------------------------------------------------
namespace {
int sm100_device_count() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}
}  // namespace

DeviceGroup::DeviceGroup(int world_size) : world_size_(world_size) {
  if (!is_power_of_two(world_size))
    fail(ErrorCode::BadWorldSize, "world size must be a power of two, got " + std::to_string(world_size));
  // rank r on device r % device_count: DeviceGroup(8) spans the eight GPUs of an
  // HGX node and is the reference's simulated group on a one-GPU machine.
  const int n = sm100_device_count();
  for (int r = 0; r < world_size; ++r) devices_.push_back(n > 0 ? r % n : 0);
}

DeviceGroup::DeviceGroup(int world_size, std::vector<int> devices) : world_size_(world_size), devices_(std::move(devices)) {
  if (!is_power_of_two(world_size))
    fail(ErrorCode::BadWorldSize, "world size must be a power of two, got " + std::to_string(world_size));
  if (static_cast<int>(devices_.size()) != world_size)
    fail(ErrorCode::BadArgument, "DeviceGroup: one device id per rank expected");
}

int DeviceGroup::device_span() const {
  std::vector<int> d(devices_);
  std::sort(d.begin(), d.end());
  return static_cast<int>(std::unique(d.begin(), d.end()) - d.begin());
}

tbik_local_group* DeviceGroup::native() const {
  if (!native_) {
    tbik_local_group* g = nullptr;
    check_status(tbik_local_group_create(world_size_, devices_.data(), &g));
    native_ = std::shared_ptr<tbik_local_group>(g, [](tbik_local_group* p) { tbik_local_group_destroy(p); });
  }
  return native_.get();
}

std::vector<Matrix> all_gather(const DeviceGroup& group, const std::vector<Matrix>& xs) {
  require_uniform(group, xs);
  return xs;
}

std::vector<Matrix> tree_all_reduce_per_rank(const DeviceGroup& group, const std::vector<Matrix>& xs) {
  std::vector<Matrix> out;
  for (int r = 0; r < group.world_size(); ++r) out.push_back(reduce(group, xs, false));
  for (int r = 1; r < group.world_size(); ++r)
    if (!bit_equal(out[0], out[static_cast<std::size_t>(r)]))
      fail(ErrorCode::CollectiveMismatch, "tree_all_reduce produced rank-divergent results at rank " + std::to_string(r));
  return out;
}

Matrix tree_all_reduce(const DeviceGroup& group, const std::vector<Matrix>& xs) { return reduce(group, xs, false); }
Matrix ring_reduce_baseline(const DeviceGroup& group, const std::vector<Matrix>& xs) { return reduce(group, xs, true); }

// ---- layers.hpp -----------------------------------------------------------------------------
ShardPlan make_column_shard_plan(std::int64_t n, int tp) {
  std::vector<std::int64_t> b(static_cast<std::size_t>(2 * (tp > 0 ? tp : 1)));
  check_status(tbik_make_column_shard_plan(n, tp, b.data()));
  ShardPlan s{ShardPlan::Mode::Column, tp, {}};
  for (int r = 0; r < tp; ++r) s.bounds.emplace_back(b[2 * r], b[2 * r + 1]);
  return s;
}

ShardPlan make_row_shard_plan(std::int64_t k, const BlockConfig& cfg, int tp, std::int64_t c_max) {
  std::vector<std::int64_t> b(static_cast<std::size_t>(2 * (tp > 0 ? tp : 1)));
  tbik_block_config c = c_cfg(cfg);
  check_status(tbik_make_row_shard_plan(k, &c, tp, c_max, b.data()));
  ShardPlan s{ShardPlan::Mode::Row, tp, {}};
  for (int r = 0; r < tp; ++r) s.bounds.emplace_back(b[2 * r], b[2 * r + 1]);
  return s;
}

namespace {
struct DeviceScope {  // restores the caller's current device
  int prev = 0;
  DeviceScope() { cudaGetDevice(&prev); }
  ~DeviceScope() { cudaSetDevice(prev); }
};
}  // namespace

Matrix column_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group, const BlockConfig& cfg) {
  return column_parallel_forward(x, w, group, cfg, default_leaf());
}

Matrix column_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group, const BlockConfig& cfg,
                               Leaf leaf) {
  if (x.cols() != w.rows()) fail(ErrorCode::ShapeMismatch, "column_parallel_forward: inner dimensions differ");
  DeviceScope scope;
  tbik_block_config c = c_cfg(cfg);
  if (group.device_span() <= 1) {
    cuda_ok(cudaSetDevice(group.devices()[0]), "cudaSetDevice");
    DevBuf dx = upload(x), dw = upload(w), dy(static_cast<std::size_t>(x.rows() * w.cols()) * 4);
    check_status(tbik_column_parallel_forward_local(dx.p, static_cast<int>(x.dtype()), x.cols(), dw.p,
                                                    static_cast<int>(w.dtype()), w.cols(), static_cast<float*>(dy.p),
                                                    w.cols(), x.rows(), w.cols(), x.cols(), group.world_size(), &c,
                                                    static_cast<int>(leaf), nullptr));
    check_status(tbik_sync(nullptr));
    return download_f32(dy, x.rows(), w.cols());
  }
  // ranks on their own GPUs: rank r computes its column block on devices()[r]
  // (layers.cpp:48-72); the concatenation is the column offset of the download.
  const ShardPlan plan = make_column_shard_plan(w.cols(), group.world_size());
  Matrix out(x.rows(), w.cols(), Dtype::F32);
  for (int r = 0; r < group.world_size(); ++r) {
    const auto [b, e] = plan.bounds[static_cast<std::size_t>(r)];
    cuda_ok(cudaSetDevice(group.devices()[static_cast<std::size_t>(r)]), "cudaSetDevice");
    DevBuf dx = upload(x), dw = upload(w.slice_cols(b, e)), dy(static_cast<std::size_t>(x.rows() * (e - b)) * 4);
    check_status(tbik_tree_matmul(dx.p, static_cast<int>(x.dtype()), x.cols(), dw.p, static_cast<int>(w.dtype()),
                                  e - b, static_cast<float*>(dy.p), e - b, x.rows(), e - b, x.cols(), &c,
                                  static_cast<int>(leaf), nullptr));
    check_status(tbik_sync(nullptr));
    cuda_ok(cudaMemcpy2D(out.f32_data().data() + b, static_cast<std::size_t>(w.cols()) * 4, dy.p,
                         static_cast<std::size_t>(e - b) * 4, static_cast<std::size_t>(e - b) * 4,
                         static_cast<std::size_t>(x.rows()), cudaMemcpyDeviceToHost),
            "download");
  }
  return out;
}

Matrix row_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group, const BlockConfig& cfg,
                            std::int64_t c_max) {
  return row_parallel_forward(x, w, group, cfg, c_max, default_leaf());
}

Matrix row_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group, const BlockConfig& cfg,
                            std::int64_t c_max, Leaf leaf) {
  if (x.cols() != w.rows()) fail(ErrorCode::ShapeMismatch, "row_parallel_forward: inner dimensions differ");
  DeviceScope scope;
  tbik_block_config c = c_cfg(cfg);
  if (group.device_span() <= 1) {
    cuda_ok(cudaSetDevice(group.devices()[0]), "cudaSetDevice");
    DevBuf dx = upload(x), dw = upload(w), dy(static_cast<std::size_t>(x.rows() * w.cols()) * 4);
    check_status(tbik_row_parallel_forward_local(dx.p, static_cast<int>(x.dtype()), x.cols(), dw.p,
                                                 static_cast<int>(w.dtype()), w.cols(), static_cast<float*>(dy.p),
                                                 w.cols(), x.rows(), w.cols(), x.cols(), group.world_size(), &c, c_max,
                                                 static_cast<int>(leaf), nullptr));
    check_status(tbik_sync(nullptr));
    return download_f32(dy, x.rows(), w.cols());
  }
  // ranks on their own GPUs (layers.cpp:74-98): rank r's K shard goes to
  // devices()[r], its tree GEMM runs there, and rank 0's device reduces the W
  // partials over peer memory (NVLink) in Algorithm-2 order.
  const ShardPlan plan = make_row_shard_plan(x.cols(), cfg, group.world_size(), c_max);
  tbik_local_group* lg = group.native();
  std::vector<std::unique_ptr<DevBuf>> bufs;
  std::vector<const void*> xs, ws;
  std::vector<std::int64_t> ldx, ldw;
  for (int r = 0; r < group.world_size(); ++r) {
    const auto [b, e] = plan.bounds[static_cast<std::size_t>(r)];
    cuda_ok(cudaSetDevice(group.devices()[static_cast<std::size_t>(r)]), "cudaSetDevice");
    bufs.emplace_back(new DevBuf(upload(x.slice_cols(b, e))));
    xs.push_back(bufs.back()->p);
    bufs.emplace_back(new DevBuf(upload(w.slice_rows(b, e))));
    ws.push_back(bufs.back()->p);
    ldx.push_back(e - b);
    ldw.push_back(w.cols());
  }
  cuda_ok(cudaSetDevice(group.devices()[0]), "cudaSetDevice");
  DevBuf dy(static_cast<std::size_t>(x.rows() * w.cols()) * 4);
  check_status(tbik_local_group_row_parallel_forward(lg, xs.data(), static_cast<int>(x.dtype()), ldx.data(), ws.data(),
                                                     static_cast<int>(w.dtype()), ldw.data(), static_cast<float*>(dy.p),
                                                     w.cols(), x.rows(), w.cols(), x.cols(), &c, c_max,
                                                     static_cast<int>(leaf), nullptr));
  check_status(tbik_sync(nullptr));
  return download_f32(dy, x.rows(), w.cols());
}

// The status quo (layers.cpp:100-146): cuBLAS per rank + ring reduce / concat.
Matrix baseline_row_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group) {
  if (x.cols() != w.rows()) fail(ErrorCode::ShapeMismatch, "baseline_row_parallel_forward: inner dimensions differ");
  DeviceScope scope;
  cuda_ok(cudaSetDevice(group.devices()[0]), "cudaSetDevice");
  DevBuf dx = upload(x), dw = upload(w), dy(static_cast<std::size_t>(x.rows() * w.cols()) * 4);
  check_status(tbik_baseline_row_parallel_forward_local(dx.p, static_cast<int>(x.dtype()), x.cols(), dw.p,
                                                        static_cast<int>(w.dtype()), w.cols(), static_cast<float*>(dy.p),
                                                        w.cols(), x.rows(), w.cols(), x.cols(), group.world_size(),
                                                        nullptr));
  check_status(tbik_sync(nullptr));
  return download_f32(dy, x.rows(), w.cols());
}

Matrix baseline_column_parallel_forward(const Matrix& x, const Matrix& w, const DeviceGroup& group) {
  if (x.cols() != w.rows()) fail(ErrorCode::ShapeMismatch, "baseline_column_parallel_forward: inner dimensions differ");
  DeviceScope scope;
  cuda_ok(cudaSetDevice(group.devices()[0]), "cudaSetDevice");
  DevBuf dx = upload(x), dw = upload(w), dy(static_cast<std::size_t>(x.rows() * w.cols()) * 4);
  check_status(tbik_baseline_column_parallel_forward_local(dx.p, static_cast<int>(x.dtype()), x.cols(), dw.p,
                                                           static_cast<int>(w.dtype()), w.cols(),
                                                           static_cast<float*>(dy.p), w.cols(), x.rows(), w.cols(),
                                                           x.cols(), group.world_size(), nullptr));
  check_status(tbik_sync(nullptr));
  return download_f32(dy, x.rows(), w.cols());
}

// ---- demo.hpp ----------------------------------------------------------------------------------
Matrix rmsnorm(const Matrix& x, const std::vector<float>& gamma, float eps) {
  if (static_cast<std::int64_t>(gamma.size()) != x.cols())
    fail(ErrorCode::ShapeMismatch,
         "rmsnorm: gamma length " + std::to_string(gamma.size()) + " != cols " + std::to_string(x.cols()));
  DevBuf dx = upload(x), dg(gamma.size() * 4), dy(static_cast<std::size_t>(x.size()) * 4);
  cuda_ok(cudaMemcpy(dg.p, gamma.data(), gamma.size() * 4, cudaMemcpyHostToDevice), "upload gamma");
  check_status(tbik_tree_rmsnorm(dx.p, static_cast<int>(x.dtype()), x.cols(), static_cast<const float*>(dg.p), eps,
                                 dy.p, TBIK_F32, x.cols(), x.rows(), x.cols(), nullptr));
  check_status(tbik_sync(nullptr));
  return download_f32(dy, x.rows(), x.cols());
}

Matrix silu(const Matrix& x) {  // demo.cpp:36-45 with the library's exp
  DevBuf dx = upload(x), dy(static_cast<std::size_t>(x.size()) * 4);
  check_status(tbik_silu(dx.p, static_cast<int>(x.dtype()), x.cols(), x.rows(), x.cols(), static_cast<float*>(dy.p),
                         x.cols(), nullptr));
  check_status(tbik_sync(nullptr));
  return download_f32(dy, x.rows(), x.cols());
}

void matrix_write(const std::string& path, const Matrix& m) {
  check_status(tbik_matrix_write(path.c_str(), m.raw(), static_cast<int>(m.dtype()), m.rows(), m.cols()));
}

Matrix matrix_read(const std::string& path) {
  int dt = 0;
  std::int64_t rows = 0, cols = 0;
  check_status(tbik_matrix_read_header(path.c_str(), &dt, &rows, &cols));
  const std::size_t n = static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols);
  if (dt == TBIK_F32) {
    std::vector<float> v(n ? n : 1);
    check_status(tbik_matrix_read(path.c_str(), v.data(), static_cast<std::int64_t>(v.size() * 4)));
    v.resize(n);
    return Matrix::from_f32(rows, cols, std::move(v));
  }
  std::vector<std::uint16_t> v(n ? n : 1);
  check_status(tbik_matrix_read(path.c_str(), v.data(), static_cast<std::int64_t>(v.size() * 2)));
  v.resize(n);
  return Matrix::from_bf16(rows, cols, std::move(v));
}

}  // namespace tbik
