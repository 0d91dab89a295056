// tbik_abi.cu -- the extern "C" boundary (include/tbik_b200.h): status
// plumbing, the integer planner (matmul.cpp:24-67, layers.cpp:9-46), launch
// dispatch, the single-device simulated DeviceGroup (the reference's
// in-process group, collective.hpp:15-23) and the one-process-per-GPU group
// over NVLink peer memory (CUDA IPC + device-side flag barrier).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <map>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tbik_common.cuh"
#include "tbik_internal.h"

namespace tbik_b200 {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}

namespace {
thread_local const char* g_last_kernel = "";
}

void count_launch(const char* kernel) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (kernel) g_last_kernel = kernel;
}

namespace {
constexpr int64_t kUnset = INT64_MIN;
std::atomic<int64_t> g_knobs[KNOB_COUNT];
struct KnobInit {
  KnobInit() {
    for (auto& k : g_knobs) k.store(kUnset);
  }
} g_knob_init;
const char* const kKnobNames[KNOB_COUNT] = {
    "tc_pair",  "tc_abox", "tc_group_m", "tc_units",       "tc_deep",         "tc_acc4",
    "tc_skinny", "sk_mt",  "sk_units",   "sk_leaf",        "sk_bn",           "fma_v1",
    "group_fused", "group_overlap", "ar_two_phase_bytes", "tc_wide", "tc_wide_tail", "sk_ks",
    "sk_pdl",    "sk_trace", "sk_pair",  "attn_sv1", "attn_tc5", "tc_pdl"};
}  // namespace

int64_t knob(Knob k, int64_t dflt) {
  const int64_t v = g_knobs[k].load(std::memory_order_relaxed);
  return v == kUnset ? dflt : v;
}

tbik_status set_error(tbik_status st, const std::string& what) {
  g_last_error = what;
  return st;
}

tbik_status cuda_status(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return TBIK_CUDA_ERROR;
}

int current_device_checked() {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  int major = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return -1;
  return major == 10 ? dev : -1;
}

namespace {
struct Arena {
  void* ptr = nullptr;
  size_t bytes = 0;
};
constexpr int kSlots = 12;
std::mutex g_ws_mu;
// (device, stream) -> slots.  std::map nodes never move, so a returned pointer
// stays valid until that same key grows the slot.
std::map<std::pair<int, uintptr_t>, std::array<Arena, kSlots>> g_ws;
}  // namespace

void* workspace(size_t bytes, int slot, cudaStream_t stream) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || slot < 0 || slot >= kSlots) return nullptr;
  std::lock_guard<std::mutex> lk(g_ws_mu);
  Arena& a = g_ws[{dev, reinterpret_cast<uintptr_t>(stream)}][slot];
  if (a.bytes >= bytes && a.ptr) return a.ptr;
  if (a.ptr) {
    cudaStreamSynchronize(stream);  // work queued on this stream may still read the old buffer
    cudaFree(a.ptr);
    a.ptr = nullptr;
    a.bytes = 0;
  }
  size_t want = std::max<size_t>(bytes, size_t(1) << 20);
  if (cudaMalloc(&a.ptr, want) != cudaSuccess) {
    a.ptr = nullptr;
    return nullptr;
  }
  a.bytes = want;
  return a.ptr;
}

// ---- planner -----------------------------------------------------------------
namespace {
bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
int64_t log2_exact(int64_t v) {
  int64_t l = 0;
  while ((int64_t{1} << l) < v) ++l;
  return l;
}
}  // namespace

// plan_blocks (matmul.cpp:24-67), identical integer semantics.
tbik_status plan(int64_t K, int64_t bk, int64_t kf_req, int64_t c_max, tbik_reduction_plan* out) {
  if (K < 1 || bk < 1) return set_error(TBIK_BAD_ARGUMENT, "plan_blocks requires K >= 1 and block_k >= 1");
  if (!is_pow2(c_max))
    return set_error(TBIK_BAD_ARGUMENT, "c_max must be a power of two, got " + std::to_string(c_max));
  const int64_t tiles = (K + bk - 1) / bk;
  auto feasible = [&](int64_t kf) {
    return kf >= 1 && tiles % kf == 0 && is_pow2(tiles / kf) && tiles / kf >= c_max;
  };
  int64_t kf = kf_req;
  if (kf == 0) {
    for (int64_t c = 1; c <= tiles; ++c)
      if (feasible(c)) {
        kf = c;
        break;
      }
    if (kf == 0)
      return set_error(TBIK_PLAN_INFEASIBLE, "no feasible k_first for K=" + std::to_string(K) +
                                                 ", block_k=" + std::to_string(bk) +
                                                 ", c_max=" + std::to_string(c_max));
  } else if (!feasible(kf)) {
    return set_error(TBIK_PLAN_INFEASIBLE, "k_first=" + std::to_string(kf) + " infeasible for K=" +
                                               std::to_string(K) + ", block_k=" + std::to_string(bk) +
                                               ", c_max=" + std::to_string(c_max));
  }
  out->tiles_total = tiles;
  out->k_first = kf;
  out->leaves = tiles / kf;
  out->depth = log2_exact(tiles / kf) + 1;
  return TBIK_OK;
}

tbik_status row_shards(int64_t K, int64_t bk, int64_t kf, int tp, int64_t c_max, int64_t* bounds) {
  if (tp > c_max)
    return set_error(TBIK_SHARD_ERROR,
                     "row shard: tp=" + std::to_string(tp) + " exceeds c_max=" + std::to_string(c_max));
  tbik_reduction_plan p;
  TBIK_TRY(plan(K, bk, kf, c_max, &p));
  if (tp < 1 || p.leaves % tp != 0)
    return set_error(TBIK_SHARD_ERROR, "row shard: " + std::to_string(p.leaves) +
                                           " leaves not divisible by tp=" + std::to_string(tp));
  const int64_t group = p.k_first * bk, per = p.leaves / tp;
  for (int r = 0; r < tp; ++r) {
    int64_t b = r * per * group, e = (r + 1) * per * group;
    if (e > K) e = K;  // ragged tail tiles live on the last rank (layers.cpp:42)
    bounds[2 * r] = b;
    bounds[2 * r + 1] = e;
  }
  return TBIK_OK;
}

// ---- dispatch -----------------------------------------------------------------
namespace {
int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}
size_t dsize(int dt) { return dt == TBIK_BF16 ? 2 : 4; }
}  // namespace

// TMA needs 16-byte row strides and base addresses.  A bf16 operand that has
// neither (any K or N not a multiple of 8) is copied once into a padded buffer
// (workspace slot `slot`, row stride rounded up to 8 elements); the padding is
// never read (the tensor map's extent is the true width), so the bits are those
// of the unpadded call.
tbik_status pad_operand(const void** p, int64_t* ld, int64_t rows, int64_t cols, int slot, cudaStream_t s) {
  const bool ok = (*ld % 8 == 0) && (reinterpret_cast<uintptr_t>(*p) & 15) == 0;
  if (ok) return TBIK_OK;
  const int64_t ldp = (cols + 7) / 8 * 8;
  void* buf = workspace(static_cast<size_t>(rows) * ldp * 2, slot, s);
  if (!buf) return set_error(TBIK_CUDA_ERROR, "tc gemm: padding buffer allocation failed");
  TBIK_CUDA(cudaMemcpy2DAsync(buf, ldp * 2, *p, *ld * 2, cols * 2, rows, cudaMemcpyDeviceToDevice, s));
  *p = buf;
  *ld = ldp;
  return TBIK_OK;
}

int64_t tc_split_units(const GemmView& v) {
  const int64_t tiles_mn = tc_tiles(v);
  // Split the K range of each output tile into 2^j aligned subtrees when it pays:
  // the split changes the wave efficiency items / (waves * slots) of the launch
  // (74 CTA pairs / 148 CTAs), and costs ~12 bytes of extra partial-output
  // traffic per output element (written by the GEMM, read + combined by
  // tree_combine_vec_kernel) against 2K flops -- about 1300 / K of the GEMM's time
  // at B200 rates.  Split while the efficiency gain exceeds that and every unit
  // keeps >= 8 leaves.  The combine continues the same tree (Theorem 1): the
  // split never changes bits.  Measured (tools/midm_sweep.py, e93, with the
  // vectorised combine): K=14336 M=768 / 2048 +9 % / +3 %, K=4096 M=256 / 768
  // +31 % / +5 % split; no split where the efficiency does not move (M=512, 1024,
  // 1536) or K is short (K=4096 M=2048: -15 % split).
  {  // 256 x 192 tiles choose their own split (tbik_gemm_tc_w192.cu)
    const int64_t w = tc_w192_units(v);
    if (w > 0 && tc_wide_variant(v) != 0) {
      int64_t units = w <= v.L && v.T / w >= 8 ? w : 1;
      const int64_t u = knob(KNOB_TC_UNITS, 0);
      if (u >= 1 && u <= v.L && (u & (u - 1)) == 0) units = u;
      return units;
    }
  }
  const int64_t slots = tc_parallel_slots(v);
  auto eff = [&](int64_t items) {
    const int64_t waves = (items + slots - 1) / slots;
    return static_cast<double>(items) / static_cast<double>(waves * slots);
  };
  int64_t units = 1;
  while (units * 2 <= v.L && v.T / (units * 2) >= 8 &&
         eff(tiles_mn * units * 2) / eff(tiles_mn * units) - 1.0 > 1300.0 / static_cast<double>(v.K) - 0.02)
    units *= 2;
  (void)next_pow2;
  {  // schedule knob tc_units (power of two <= leaves; same bits)
    const int64_t u = knob(KNOB_TC_UNITS, 0);
    if (u >= 1 && u <= v.L && (u & (u - 1)) == 0) units = u;
  }
  return units;
}

tbik_status run_tree_gemm(const GemmView& v, float* C, int64_t ldc, int leaf_mode, cudaStream_t s) {
  const size_t slice = static_cast<size_t>(v.M) * v.N;
  if (leaf_mode == TBIK_LEAF_TCGEN05) {
    if (tc_use_skinny(v)) {
      const tbik_status st = launch_tc_skinny(v, C, ldc, s);
      if (st != TBIK_UNSUPPORTED) return st;
    }
    const int64_t units = tc_split_units(v);
    if (units <= 1) {
      GemmOut o{OUT_FULL, v.T, C, ldc, 0};
      return launch_tc_gemm(v, o, s);
    }
    float* ws = static_cast<float*>(workspace(slice * units * sizeof(float), 0, s));
    if (!ws) return set_error(TBIK_CUDA_ERROR, "workspace allocation failed");
    GemmOut o{OUT_UNITS, v.T / units, ws, v.N, static_cast<int64_t>(slice)};
    TBIK_TRY(launch_tc_gemm(v, o, s));
    return launch_tree_combine(ws, units, 1, v.M, v.N, C, ldc, s);
  }
  if (leaf_mode != TBIK_LEAF_FMA) return set_error(TBIK_BAD_ARGUMENT, "unknown leaf mode");
  const bool leaves = v.M <= 64 && slice * v.T * sizeof(float) <= (size_t(1) << 28);
  const int64_t X = leaves ? v.T : v.L;
  float* ws = static_cast<float*>(workspace(slice * X * sizeof(float), 0, s));
  if (!ws) return set_error(TBIK_CUDA_ERROR, "workspace allocation failed");
  GemmOut o{leaves ? OUT_LEAVES : OUT_GROUPS, leaves ? 1 : v.kf, ws, v.N, static_cast<int64_t>(slice)};
  TBIK_TRY(launch_fma_gemm(v, o, s));
  return launch_tree_combine(ws, X, leaves ? v.kf : 1, v.M, v.N, C, ldc, s);
}

tbik_status make_view(const void* A, int adt, int64_t lda, const void* B, int bdt, int64_t ldb, int64_t M,
                      int64_t N, int64_t K, int64_t bk, int64_t kf_global, GemmView* v) {
  // Local plan of this view with the given (global) k_first, c_max = 1
  // (matmul.cpp:153 via layers.cpp:85-88).
  tbik_reduction_plan p;
  TBIK_TRY(plan(K, bk, kf_global, 1, &p));
  *v = GemmView{A, adt, lda, B, bdt, ldb, M, N, K, bk, p.k_first, p.tiles_total, p.leaves};
  return TBIK_OK;
}

namespace {

tbik_status check_mat(const void* p, int dt, int64_t rows, int64_t cols, int64_t ld, const char* name) {
  if (rows < 1 || cols < 1)
    return set_error(TBIK_BAD_DIMENSION, std::string(name) + ": dimensions must be >= 1");
  if (dt != TBIK_F32 && dt != TBIK_BF16) return set_error(TBIK_UNKNOWN_DTYPE, std::string(name) + ": dtype");
  if (ld < cols) return set_error(TBIK_BAD_ARGUMENT, std::string(name) + ": leading dimension < cols");
  if (!p) return set_error(TBIK_BAD_ARGUMENT, std::string(name) + ": null pointer");
  return TBIK_OK;
}

tbik_status require_device() {
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 CUDA device (no CPU fallback)");
  return TBIK_OK;
}

}  // namespace

}  // namespace tbik_b200

using namespace tbik_b200;

// ============================================================================
// extern "C"
// ============================================================================
extern "C" {

const char* tbik_status_string(int st) {
  switch (st) {
    case TBIK_OK: return "ok";
    case TBIK_BAD_DIMENSION: return "BadDimension";
    case TBIK_SHAPE_MISMATCH: return "ShapeMismatch";
    case TBIK_BAD_MAGIC: return "BadMagic";
    case TBIK_TRUNCATED: return "Truncated";
    case TBIK_UNKNOWN_DTYPE: return "UnknownDtype";
    case TBIK_PLAN_INFEASIBLE: return "PlanInfeasible";
    case TBIK_SHARD_ERROR: return "ShardError";
    case TBIK_BAD_WORLD_SIZE: return "BadWorldSize";
    case TBIK_COLLECTIVE_MISMATCH: return "CollectiveMismatch";
    case TBIK_BAD_ARGUMENT: return "BadArgument";
    case TBIK_IO: return "Io";
    case TBIK_CUDA_ERROR: return "CudaError";
    case TBIK_NO_DEVICE: return "NoDevice";
    case TBIK_UNSUPPORTED: return "Unsupported";
    default: return "unknown";
  }
}

const char* tbik_last_error(void) { return g_last_error.c_str(); }
tbik_status tbik_set_schedule(const char* name, int64_t value) {
  if (!name) {  // NULL: clear every override
    for (auto& k : g_knobs) k.store(kUnset);
    return TBIK_OK;
  }
  for (int i = 0; i < KNOB_COUNT; ++i)
    if (std::strcmp(name, kKnobNames[i]) == 0) {
      g_knobs[i].store(value < 0 ? kUnset : value);
      return TBIK_OK;
    }
  return set_error(TBIK_BAD_ARGUMENT, std::string("unknown schedule knob '") + name + "'");
}

int tbik_version(void) { return 100; }
uint64_t tbik_launch_count(void) { return g_launches.load(); }
const char* tbik_last_kernel(void) { return tbik_b200::g_last_kernel; }

int tbik_device_available(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) return 0;
  return current_device_checked() >= 0 ? 1 : 0;
}

tbik_status tbik_sync(void* stream) {
  TBIK_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  TBIK_CUDA(cudaGetLastError());
  return TBIK_OK;
}

tbik_status tbik_default_block_config(int dtype, tbik_block_config* out) {
  if (!out) return set_error(TBIK_BAD_ARGUMENT, "null out");
  if (dtype == TBIK_BF16)
    *out = tbik_block_config{64, 256, 128, 0};  // matmul.cpp:12
  else if (dtype == TBIK_F32)
    *out = tbik_block_config{32, 128, 64, 0};  // matmul.cpp:13
  else
    return set_error(TBIK_UNKNOWN_DTYPE, "unknown dtype");
  return TBIK_OK;
}

tbik_status tbik_plan_blocks(int64_t K, const tbik_block_config* cfg, int64_t c_max, tbik_reduction_plan* out) {
  if (!cfg || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  return plan(K, cfg->block_k, cfg->k_first, c_max, out);
}

tbik_status tbik_make_row_shard_plan(int64_t K, const tbik_block_config* cfg, int tp, int64_t c_max,
                                     int64_t* bounds) {
  if (!cfg || !bounds) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  return row_shards(K, cfg->block_k, cfg->k_first, tp, c_max, bounds);
}

tbik_status tbik_make_column_shard_plan(int64_t N, int tp, int64_t* bounds) {
  if (!bounds) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (tp < 1 || N % tp != 0)  // layers.cpp:10-15
    return set_error(TBIK_SHARD_ERROR, "column shard: N=" + std::to_string(N) + " not divisible by tp=" +
                                           std::to_string(tp));
  const int64_t w = N / tp;
  for (int r = 0; r < tp; ++r) {
    bounds[2 * r] = r * w;
    bounds[2 * r + 1] = (r + 1) * w;
  }
  return TBIK_OK;
}

tbik_status tbik_tree_matmul(const void* A, int a_dtype, int64_t lda, const void* B, int b_dtype, int64_t ldb,
                             float* C, int64_t ldc, int64_t M, int64_t N, int64_t K, const tbik_block_config* cfg,
                             int leaf_mode, void* stream) {
  if (!cfg) return set_error(TBIK_BAD_ARGUMENT, "null cfg");
  TBIK_TRY(check_mat(A, a_dtype, M, K, lda, "A"));
  TBIK_TRY(check_mat(B, b_dtype, K, N, ldb, "B"));
  TBIK_TRY(check_mat(C, TBIK_F32, M, N, ldc, "C"));
  if (cfg->block_m < 1 || cfg->block_n < 1 || cfg->block_k < 1)
    return set_error(TBIK_BAD_ARGUMENT, "block sizes must be >= 1");  // matmul.cpp:150-152
  TBIK_TRY(require_device());
  GemmView v;
  TBIK_TRY(make_view(A, a_dtype, lda, B, b_dtype, ldb, M, N, K, cfg->block_k, cfg->k_first, &v));
  return run_tree_gemm(v, C, ldc, leaf_mode, static_cast<cudaStream_t>(stream));
}

tbik_status tbik_tree_matmul_silu_mul(const void* A, int a_dtype, int64_t lda, const void* B, int b_dtype,
                                      int64_t ldb, void* act, int64_t ld_act, int64_t M, int64_t I, int64_t K,
                                      const tbik_block_config* cfg, int leaf_mode, void* stream) {
  if (!cfg || !act) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (I < 1) return set_error(TBIK_BAD_DIMENSION, "silu_mul: inter must be >= 1");
  const int64_t N = 2 * I;
  TBIK_TRY(check_mat(A, a_dtype, M, K, lda, "A"));
  TBIK_TRY(check_mat(B, b_dtype, K, N, ldb, "B"));
  if (ld_act < I) return set_error(TBIK_BAD_ARGUMENT, "act: leading dimension < inter");
  TBIK_TRY(require_device());
  GemmView v;
  TBIK_TRY(make_view(A, a_dtype, lda, B, b_dtype, ldb, M, N, K, cfg->block_k, cfg->k_first, &v));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // SiLU*up in the wide GEMM's epilogue; decode sizes (M <= 128) go through the
  // skinny weight-streaming kernel instead (the separate SiLU*up pass over M x N
  // f32 is small there), same bits either way.
  if (leaf_mode == TBIK_LEAF_TCGEN05 && !tc_use_skinny(v) && tc_split_units(v) <= 1) {
    GemmOut o{OUT_FULL, v.T, nullptr, N, 0, static_cast<uint16_t*>(act), ld_act};
    return launch_tc_gemm(v, o, s);
  }
  // split launches / exact leaf: f32 tree GEMM, then the same SiLU*up as a kernel
  float* tmp = static_cast<float*>(workspace(static_cast<size_t>(M) * N * sizeof(float), 10, s));
  if (!tmp) return set_error(TBIK_CUDA_ERROR, "workspace allocation failed");
  TBIK_TRY(run_tree_gemm(v, tmp, N, leaf_mode, s));
  return launch_silu_mul_il(tmp, N, M, I, static_cast<uint16_t*>(act), ld_act, s);
}

tbik_status tbik_tree_matmul_logits(const void* A, int a_dtype, int64_t lda, const void* B, int b_dtype, int64_t ldb,
                                    float* C, int64_t ldc, float* chunk_ms, int64_t ld_chunks, int64_t M, int64_t N,
                                    int64_t K, int64_t groups, const tbik_block_config* cfg, int leaf_mode,
                                    void* stream) {
  if (!cfg || !chunk_ms) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  TBIK_TRY(check_mat(A, a_dtype, M, K, lda, "A"));
  TBIK_TRY(check_mat(B, b_dtype, K, N, ldb, "B"));
  TBIK_TRY(check_mat(C, TBIK_F32, M, N, ldc, "C"));
  if (groups < 1 || (groups & (groups - 1)) || N % groups)
    return set_error(TBIK_SHARD_ERROR, "logits: groups must be a power of two dividing N");
  TBIK_TRY(require_device());
  GemmView v;
  TBIK_TRY(make_view(A, a_dtype, lda, B, b_dtype, ldb, M, N, K, cfg->block_k, cfg->k_first, &v));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n = N / groups, nc = (n + 15) / 16;
  if (ld_chunks < groups * nc) return set_error(TBIK_BAD_ARGUMENT, "logits: ld_chunks < groups * chunks per group");
  // The chunk states come out of the 256x128 tcgen05 GEMM's epilogue when the GEMM is
  // one FULL pair-tile launch (M > 128; not the skinny or K-split schedules, and not a
  // shape where the 256x192 kernel is the default: its plain GEMM + a pass over the
  // logits measured faster than the 256x128 epilogue, tools/lm_head_w192.py) and chunks
  // are absolute 16-column blocks (n % 16 == 0); otherwise a pass over the logits
  // computes the same states (tb_ms_chunk16 in both) -- a pure scheduling choice.
  if (leaf_mode == TBIK_LEAF_TCGEN05 && n % 16 == 0 && M > 128 && !tc_use_skinny(v) && tc_split_units(v) <= 1 &&
      tc_wide_variant(v) == 0 && tc_supported(v, nullptr) && (reinterpret_cast<uintptr_t>(chunk_ms) & 7) == 0) {
    GemmOut o{OUT_FULL, v.T, C, ldc, 0};
    o.ms = chunk_ms;
    o.ld_ms = 2 * ld_chunks;
    return launch_tc_gemm(v, o, s);
  }
  TBIK_TRY(run_tree_gemm(v, C, ldc, leaf_mode, s));
  return tbik_logsoftmax_chunk_states(C, ldc, M, N, groups, chunk_ms, ld_chunks, stream);
}

tbik_status tbik_tree_matmul_leaves(const void* A, int a_dtype, int64_t lda, const void* B, int b_dtype,
                                    int64_t ldb, float* leaves, int64_t M, int64_t N, int64_t K,
                                    const tbik_block_config* cfg, int leaf_mode, void* stream) {
  if (!cfg) return set_error(TBIK_BAD_ARGUMENT, "null cfg");
  TBIK_TRY(check_mat(A, a_dtype, M, K, lda, "A"));
  TBIK_TRY(check_mat(B, b_dtype, K, N, ldb, "B"));
  if (!leaves) return set_error(TBIK_BAD_ARGUMENT, "null leaves");
  TBIK_TRY(require_device());
  GemmView v;
  TBIK_TRY(make_view(A, a_dtype, lda, B, b_dtype, ldb, M, N, K, cfg->block_k, cfg->k_first, &v));
  GemmOut o{OUT_LEAVES, 1, leaves, N, M * N};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (leaf_mode == TBIK_LEAF_TCGEN05) return launch_tc_gemm(v, o, s);
  if (leaf_mode == TBIK_LEAF_FMA) return launch_fma_gemm(v, o, s);
  return set_error(TBIK_BAD_ARGUMENT, "unknown leaf mode");
}

tbik_status tbik_tree_all_reduce_local(const float* const* partials, int W, float* out, int64_t elems,
                                       void* stream) {
  if (!is_pow2(W))  // DeviceGroup (collective.cpp:11-16)
    return set_error(TBIK_BAD_WORLD_SIZE, "world size must be a power of two, got " + std::to_string(W));
  if (W > kMaxRanks) return set_error(TBIK_BAD_WORLD_SIZE, "world size too large");
  if (!partials || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  TBIK_TRY(require_device());
  PartPtrs pp{};
  bool aligned = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (int r = 0; r < W; ++r) {
    if (!partials[r]) return set_error(TBIK_COLLECTIVE_MISMATCH, "null contribution from rank " + std::to_string(r));
    pp.p[r] = partials[r];
    aligned = aligned && (reinterpret_cast<uintptr_t>(partials[r]) & 15) == 0;
  }
  return launch_allreduce(pp, W, out, elems, false, aligned, static_cast<cudaStream_t>(stream));
}

tbik_status tbik_ring_reduce_local(const float* const* partials, int W, float* out, int64_t elems, void* stream) {
  if (!is_pow2(W)) return set_error(TBIK_BAD_WORLD_SIZE, "world size must be a power of two");
  if (W > 8) return set_error(TBIK_BAD_WORLD_SIZE, "ring baseline supports W <= 8");
  if (!partials || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  TBIK_TRY(require_device());
  PartPtrs pp{};
  bool aligned = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (int r = 0; r < W; ++r) {
    pp.p[r] = partials[r];
    aligned = aligned && (reinterpret_cast<uintptr_t>(partials[r]) & 15) == 0;
  }
  return launch_allreduce(pp, W, out, elems, true, aligned, static_cast<cudaStream_t>(stream));
}

tbik_status tbik_column_parallel_forward_local(const void* X, int x_dtype, int64_t ldx, const void* W, int w_dtype,
                                               int64_t ldw, float* Y, int64_t ldy, int64_t M, int64_t N, int64_t K,
                                               int tp, const tbik_block_config* cfg, int leaf_mode, void* stream) {
  if (!cfg) return set_error(TBIK_BAD_ARGUMENT, "null cfg");
  TBIK_TRY(check_mat(X, x_dtype, M, K, ldx, "X"));
  TBIK_TRY(check_mat(W, w_dtype, K, N, ldw, "W"));
  TBIK_TRY(check_mat(Y, TBIK_F32, M, N, ldy, "Y"));
  if (!is_pow2(tp)) return set_error(TBIK_BAD_WORLD_SIZE, "world size must be a power of two");
  int64_t bounds[2 * kMaxRanks];
  if (tp > kMaxRanks) return set_error(TBIK_BAD_WORLD_SIZE, "world size too large");
  TBIK_TRY(tbik_make_column_shard_plan(N, tp, bounds));
  TBIK_TRY(require_device());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int r = 0; r < tp; ++r) {
    const int64_t b = bounds[2 * r], e = bounds[2 * r + 1];
    GemmView v;
    const void* Wr = static_cast<const char*>(W) + b * dsize(w_dtype);
    TBIK_TRY(make_view(X, x_dtype, ldx, Wr, w_dtype, ldw, M, e - b, K, cfg->block_k, cfg->k_first, &v));
    TBIK_TRY(run_tree_gemm(v, Y + b, ldy, leaf_mode, s));  // concatenation = column offset
  }
  return TBIK_OK;
}

tbik_status tbik_row_parallel_forward_local(const void* X, int x_dtype, int64_t ldx, const void* W, int w_dtype,
                                            int64_t ldw, float* Y, int64_t ldy, int64_t M, int64_t N, int64_t K,
                                            int tp, const tbik_block_config* cfg, int64_t c_max, int leaf_mode,
                                            void* stream) {
  if (!cfg) return set_error(TBIK_BAD_ARGUMENT, "null cfg");
  TBIK_TRY(check_mat(X, x_dtype, M, K, ldx, "X"));
  TBIK_TRY(check_mat(W, w_dtype, K, N, ldw, "W"));
  TBIK_TRY(check_mat(Y, TBIK_F32, M, N, ldy, "Y"));
  if (!is_pow2(tp)) return set_error(TBIK_BAD_WORLD_SIZE, "world size must be a power of two, got " + std::to_string(tp));
  if (tp > kMaxRanks) return set_error(TBIK_BAD_WORLD_SIZE, "world size too large");
  int64_t bounds[2 * kMaxRanks];
  TBIK_TRY(row_shards(K, cfg->block_k, cfg->k_first, tp, c_max, bounds));
  tbik_reduction_plan gp;
  TBIK_TRY(plan(K, cfg->block_k, cfg->k_first, c_max, &gp));
  TBIK_TRY(require_device());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (tp == 1) {
    GemmView v;
    TBIK_TRY(make_view(X, x_dtype, ldx, W, w_dtype, ldw, M, N, K, cfg->block_k, gp.k_first, &v));
    return run_tree_gemm(v, Y, ldy, leaf_mode, s);
  }
  const size_t slice = static_cast<size_t>(M) * N;
  const size_t pitch = (slice + 3) & ~size_t(3);  // keep every partial 16-byte aligned
  float* parts = static_cast<float*>(workspace(pitch * tp * sizeof(float), 2, s));
  if (!parts) return set_error(TBIK_CUDA_ERROR, "partials allocation failed");
  PartPtrs pp{};
  for (int r = 0; r < tp; ++r) {
    const int64_t b = bounds[2 * r], e = bounds[2 * r + 1];
    const void* Xr = static_cast<const char*>(X) + b * dsize(x_dtype);
    const void* Wr = static_cast<const char*>(W) + b * ldw * dsize(w_dtype);
    GemmView v;
    // Every rank uses the GLOBAL k_first (layers.cpp:85-88).
    TBIK_TRY(make_view(Xr, x_dtype, ldx, Wr, w_dtype, ldw, M, N, e - b, cfg->block_k, gp.k_first, &v));
    TBIK_TRY(run_tree_gemm(v, parts + pitch * r, N, leaf_mode, s));
    pp.p[r] = parts + pitch * r;
  }
  if (ldy == N) return launch_allreduce(pp, tp, Y, static_cast<int64_t>(slice), false, (reinterpret_cast<uintptr_t>(Y) & 15) == 0, s);
  float* tmp = static_cast<float*>(workspace(slice * sizeof(float), 3, s));
  if (!tmp) return set_error(TBIK_CUDA_ERROR, "allocation failed");
  TBIK_TRY(launch_allreduce(pp, tp, tmp, static_cast<int64_t>(slice), false, true, s));
  TBIK_CUDA(cudaMemcpy2DAsync(Y, ldy * sizeof(float), tmp, N * sizeof(float), N * sizeof(float), M,
                              cudaMemcpyDeviceToDevice, s));
  return TBIK_OK;
}

}  // extern "C"

extern "C" int tbik_debug_tc_stats(unsigned long long* out, int max) { return tbik_b200::tc_debug_stats(out, max); }
