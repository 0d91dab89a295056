// tbik_local.cu -- the reference's in-process DeviceGroup on several GPUs
// (collective.hpp:15-23, layers.cpp:74-98), the small scalar entry points of
// the drop-in API (leaf_dot, matmul.cpp:69-75; silu, demo.cpp:36-45), and the
// labelled non-invariant status-quo layers (cuBLAS + ring / NCCL,
// collective.cpp:94-106, layers.cpp:100-146).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tbik_common.cuh"
#include "tbik_internal.h"
#include "tbik_mathfn.cuh"

struct tbik_local_group {
  int W = 0;
  int dev[tbik_b200::kMaxRanks] = {};
  // Ranks that share a device share the stream of the first of them: the launchers'
  // per-device workspaces are then never used by two streams at once.
  int owner[tbik_b200::kMaxRanks] = {};
  cudaStream_t stream[tbik_b200::kMaxRanks] = {};
  cudaEvent_t done[tbik_b200::kMaxRanks] = {};
  cudaEvent_t start[tbik_b200::kMaxRanks] = {};  // one per distinct-device slot (indexed by rank)
  float* part[tbik_b200::kMaxRanks] = {};
  size_t part_bytes[tbik_b200::kMaxRanks] = {};
};

namespace tbik_b200 {
namespace {

// leaf_dot (matmul.cpp:69-75): acc = fma(a[k], b[k], acc) for k ascending from +0.
__global__ void leaf_dot_kernel(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                                float* __restrict__ out) {
  float acc = 0.0f;
  for (int64_t k = 0; k < n; ++k) acc = __fmaf_rn(a[k], b[k], acc);
  *out = acc;
}

template <typename TX>
__global__ void silu_kernel(const TX* __restrict__ x, int64_t ldx, int64_t cols, float* __restrict__ out,
                            int64_t ldo) {
  const int64_t row = blockIdx.y;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float z = load_as_f32(x + row * ldx + j);
    out[row * ldo + j] = __fdiv_rn(z, __fadd_rn(1.0f, tb_exp(-z)));  // the shared exp (tbik_mathfn.cuh)
  }
}

// ring_reduce_baseline order (collective.cpp:94-106): ((p0 + p1) + p2) + ...
__global__ void ring_sum_kernel(PartPtrs parts, int W, int64_t rows, int64_t cols, float* __restrict__ out,
                                int64_t ldo) {
  const int64_t n = rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = parts.p[0][i];
    for (int r = 1; r < W; ++r) acc = __fadd_rn(acc, parts.p[r][i]);
    out[(i / cols) * ldo + i % cols] = acc;
  }
}

// ---- cuBLAS (one handle per device; calls serialised per device) ----------------
std::mutex g_blas_mu;
cublasHandle_t g_blas[16] = {};

tbik_status blas_gemm(const void* A, int adt, int64_t lda, const void* B, int bdt, int64_t ldb, void* C, int cdt,
                      int64_t ldc, int64_t M, int64_t N, int64_t K, cudaStream_t s) {
  int dev = 0;
  TBIK_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) return set_error(TBIK_UNSUPPORTED, "device index >= 16");
  if (adt != bdt) return set_error(TBIK_UNKNOWN_DTYPE, "baseline gemm: A and B must share a dtype");
  std::lock_guard<std::mutex> lk(g_blas_mu);
  if (!g_blas[dev] && cublasCreate(&g_blas[dev]) != CUBLAS_STATUS_SUCCESS)
    return set_error(TBIK_CUDA_ERROR, "cublasCreate failed");
  cublasHandle_t h = g_blas[dev];
  cublasSetStream(h, s);
  const float one = 1.0f, zero = 0.0f;
  const cudaDataType_t ab = adt == TBIK_BF16 ? CUDA_R_16BF : CUDA_R_32F;
  const cudaDataType_t ct = cdt == TBIK_BF16 ? CUDA_R_16BF : CUDA_R_32F;
  // Row-major C = A B  <=>  column-major C^T = B^T A^T.
  const cublasStatus_t st =
      cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(N), static_cast<int>(M), static_cast<int>(K), &one,
                   B, ab, static_cast<int>(ldb), A, ab, static_cast<int>(lda), &zero, C, ct, static_cast<int>(ldc),
                   CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  if (st != CUBLAS_STATUS_SUCCESS) return set_error(TBIK_CUDA_ERROR, "cublasGemmEx failed: " + std::to_string(st));
  return TBIK_OK;
}

tbik_status check_dense(const void* p, int dt, int64_t rows, int64_t cols, int64_t ld, const char* name) {
  if (!p) return set_error(TBIK_BAD_ARGUMENT, std::string(name) + ": null pointer");
  if (rows < 1 || cols < 1) return set_error(TBIK_BAD_DIMENSION, std::string(name) + ": dimensions must be >= 1");
  if (dt != TBIK_F32 && dt != TBIK_BF16) return set_error(TBIK_UNKNOWN_DTYPE, std::string(name) + ": dtype");
  if (ld < cols) return set_error(TBIK_BAD_ARGUMENT, std::string(name) + ": leading dimension < cols");
  if (rows > 0x7FFFFFFF || cols > 0x7FFFFFFF || ld > 0x7FFFFFFF)
    return set_error(TBIK_UNSUPPORTED, std::string(name) + ": dimension exceeds int32");
  return TBIK_OK;
}

size_t esize(int dt) { return dt == TBIK_BF16 ? 2 : 4; }

}  // namespace
}  // namespace tbik_b200

using namespace tbik_b200;

extern "C" {

tbik_status tbik_leaf_dot(const float* a, const float* b, int64_t n, float* out, void* stream) {
  if (!out || (n > 0 && (!a || !b))) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (n < 0) return set_error(TBIK_BAD_DIMENSION, "leaf_dot: n must be >= 0");
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  leaf_dot_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(a, b, n, out);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_silu(const void* x, int x_dtype, int64_t ldx, int64_t rows, int64_t cols, float* out, int64_t ldo,
                      void* stream) {
  TBIK_TRY(check_dense(x, x_dtype, rows, cols, ldx, "x"));
  TBIK_TRY(check_dense(out, TBIK_F32, rows, cols, ldo, "out"));
  if (rows > 65535) return set_error(TBIK_UNSUPPORTED, "silu: > 65535 rows per call");
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((cols + 255) / 256, 64)), static_cast<unsigned>(rows));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (x_dtype == TBIK_BF16)
    silu_kernel<uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(x), ldx, cols, out, ldo);
  else
    silu_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), ldx, cols, out, ldo);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

// ---- single-process multi-device group ------------------------------------------
tbik_status tbik_local_group_create(int world_size, const int* device_ids, tbik_local_group** out) {
  if (!out || !device_ids) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (world_size < 1 || (world_size & (world_size - 1)) || world_size > kMaxRanks)
    return set_error(TBIK_BAD_WORLD_SIZE, "world size must be a power of two <= 64, got " + std::to_string(world_size));
  int ndev = 0;
  TBIK_CUDA(cudaGetDeviceCount(&ndev));
  int prev = 0;
  TBIK_CUDA(cudaGetDevice(&prev));
  auto* g = new tbik_local_group();
  g->W = world_size;
  tbik_status st = TBIK_OK;
  for (int r = 0; r < world_size && st == TBIK_OK; ++r) {
    const int d = device_ids[r];
    if (d < 0 || d >= ndev) {
      st = set_error(TBIK_BAD_ARGUMENT, "device id " + std::to_string(d) + " out of range");
      break;
    }
    g->dev[r] = d;
    if (cudaSetDevice(d) != cudaSuccess || current_device_checked() < 0) {
      st = set_error(TBIK_NO_DEVICE, "device " + std::to_string(d) + " is not an sm_100 device");
      break;
    }
    g->owner[r] = r;
    for (int q = 0; q < r; ++q)
      if (g->dev[q] == d) {
        g->owner[r] = q;
        break;
      }
    if (g->owner[r] == r && cudaStreamCreateWithFlags(&g->stream[r], cudaStreamNonBlocking) != cudaSuccess)
      st = set_error(TBIK_CUDA_ERROR, "stream creation failed");
    else if (g->owner[r] != r)
      g->stream[r] = g->stream[g->owner[r]];
    if (st != TBIK_OK) break;
    if (cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->start[r], cudaEventDisableTiming) != cudaSuccess)
      st = set_error(TBIK_CUDA_ERROR, "stream / event creation failed");
  }
  // rank 0's device reads every partial: peer access from it to each other device
  if (st == TBIK_OK) {
    cudaSetDevice(g->dev[0]);
    for (int r = 1; r < world_size && st == TBIK_OK; ++r) {
      if (g->dev[r] == g->dev[0]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, g->dev[0], g->dev[r]);
      if (!can) {
        st = set_error(TBIK_UNSUPPORTED, "no peer access between devices " + std::to_string(g->dev[0]) + " and " +
                                             std::to_string(g->dev[r]));
        break;
      }
      const cudaError_t e = cudaDeviceEnablePeerAccess(g->dev[r], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else if (e != cudaSuccess)
        st = cuda_status(e, "cudaDeviceEnablePeerAccess");
    }
  }
  cudaSetDevice(prev);
  if (st != TBIK_OK) {
    tbik_local_group_destroy(g);
    return st;
  }
  *out = g;
  return TBIK_OK;
}

tbik_status tbik_local_group_destroy(tbik_local_group* g) {
  if (!g) return TBIK_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  for (int r = 0; r < g->W; ++r) {  // shared streams belong to their owner rank only
    cudaSetDevice(g->dev[r]);
    if (g->stream[r] && g->owner[r] == r) cudaStreamSynchronize(g->stream[r]);
  }
  for (int r = 0; r < g->W; ++r) {
    cudaSetDevice(g->dev[r]);
    if (g->part[r]) cudaFree(g->part[r]);
    if (g->stream[r] && g->owner[r] == r) cudaStreamDestroy(g->stream[r]);
    if (g->done[r]) cudaEventDestroy(g->done[r]);
    if (g->start[r]) cudaEventDestroy(g->start[r]);
  }
  cudaSetDevice(prev);
  delete g;
  return TBIK_OK;
}

int tbik_local_group_device(const tbik_local_group* g, int rank) {
  return g && rank >= 0 && rank < g->W ? g->dev[rank] : -1;
}

void* tbik_local_group_stream(const tbik_local_group* g, int rank) {
  return g && rank >= 0 && rank < g->W ? static_cast<void*>(g->stream[rank]) : nullptr;
}

tbik_status tbik_local_group_row_parallel_forward(tbik_local_group* g, const void* const* X_shards, int x_dtype,
                                                  const int64_t* ldx, const void* const* W_shards, int w_dtype,
                                                  const int64_t* ldw, float* Y, int64_t ldy, int64_t M, int64_t N,
                                                  int64_t K_global, const tbik_block_config* cfg, int64_t c_max,
                                                  int leaf_mode, void* stream) {
  if (!g || !X_shards || !W_shards || !ldx || !ldw || !Y || !cfg) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (M < 1 || N < 1) return set_error(TBIK_BAD_DIMENSION, "dimensions must be >= 1");
  if (ldy < N) return set_error(TBIK_BAD_ARGUMENT, "Y: leading dimension < N");
  int64_t bounds[2 * kMaxRanks];
  TBIK_TRY(tbik_make_row_shard_plan(K_global, cfg, g->W, c_max, bounds));
  tbik_reduction_plan gp;
  TBIK_TRY(tbik_plan_blocks(K_global, cfg, c_max, &gp));
  tbik_block_config local = *cfg;
  local.k_first = gp.k_first;  // layers.cpp:85-88
  int prev = 0;
  TBIK_CUDA(cudaGetDevice(&prev));
  cudaStream_t s0 = static_cast<cudaStream_t>(stream);
  const size_t bytes = static_cast<size_t>(M) * N * sizeof(float);
  tbik_status st = TBIK_OK;
  // The caller's stream on rank 0's device orders the group's work after earlier
  // work there; the other devices' inputs are ordered on their rank streams.
  if (cudaSetDevice(g->dev[0]) != cudaSuccess || cudaEventRecord(g->start[0], s0) != cudaSuccess)
    st = set_error(TBIK_CUDA_ERROR, "event record");
  PartPtrs pp{};
  for (int r = 0; r < g->W && st == TBIK_OK; ++r) {
    if (cudaSetDevice(g->dev[r]) != cudaSuccess) {
      st = set_error(TBIK_CUDA_ERROR, "cudaSetDevice");
      break;
    }
    if (g->part_bytes[r] < bytes) {  // grow (never inside a capture)
      cudaStreamSynchronize(g->stream[r]);
      if (g->part[r]) cudaFree(g->part[r]);
      g->part[r] = nullptr;
      g->part_bytes[r] = 0;
      if (cudaMalloc(&g->part[r], bytes) != cudaSuccess) {
        st = set_error(TBIK_CUDA_ERROR, "partial allocation failed");
        break;
      }
      g->part_bytes[r] = bytes;
    }
    if (g->owner[r] == r && g->dev[r] == g->dev[0] && cudaStreamWaitEvent(g->stream[r], g->start[0], 0) != cudaSuccess) {
      st = set_error(TBIK_CUDA_ERROR, "stream wait");
      break;
    }
    const int64_t Kr = bounds[2 * r + 1] - bounds[2 * r];
    st = tbik_tree_matmul(X_shards[r], x_dtype, ldx[r], W_shards[r], w_dtype, ldw[r], g->part[r], N, M, N, Kr, &local,
                          leaf_mode, g->stream[r]);
    if (st == TBIK_OK && cudaEventRecord(g->done[r], g->stream[r]) != cudaSuccess)
      st = set_error(TBIK_CUDA_ERROR, "event record");
    pp.p[r] = g->part[r];
  }
  if (st == TBIK_OK && cudaSetDevice(g->dev[0]) != cudaSuccess) st = set_error(TBIK_CUDA_ERROR, "cudaSetDevice");
  for (int r = 0; r < g->W && st == TBIK_OK; ++r)
    if (cudaStreamWaitEvent(s0, g->done[r], 0) != cudaSuccess) st = set_error(TBIK_CUDA_ERROR, "stream wait");
  if (st == TBIK_OK) {
    // Algorithm 2 over the W partials, read over peer memory by rank 0's device.
    if (ldy == N) {
      st = launch_allreduce(pp, g->W, Y, M * N, false, (reinterpret_cast<uintptr_t>(Y) & 15) == 0, s0);
    } else {
      float* tmp = static_cast<float*>(workspace(bytes, 3, s0));
      st = tmp ? launch_allreduce(pp, g->W, tmp, M * N, false, true, s0)
               : set_error(TBIK_CUDA_ERROR, "workspace allocation failed");
      if (st == TBIK_OK && cudaMemcpy2DAsync(Y, ldy * 4, tmp, N * 4, N * 4, M, cudaMemcpyDeviceToDevice, s0) != cudaSuccess)
        st = set_error(TBIK_CUDA_ERROR, "copy");
    }
  }
  cudaSetDevice(prev);
  return st;
}

// ---- the non-invariant status quo --------------------------------------------------
tbik_status tbik_baseline_gemm(const void* A, int a_dtype, int64_t lda, const void* B, int b_dtype, int64_t ldb,
                               float* C, int64_t ldc, int64_t M, int64_t N, int64_t K, void* stream) {
  TBIK_TRY(check_dense(A, a_dtype, M, K, lda, "A"));
  TBIK_TRY(check_dense(B, b_dtype, K, N, ldb, "B"));
  TBIK_TRY(check_dense(C, TBIK_F32, M, N, ldc, "C"));
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  return blas_gemm(A, a_dtype, lda, B, b_dtype, ldb, C, TBIK_F32, ldc, M, N, K, static_cast<cudaStream_t>(stream));
}

tbik_status tbik_baseline_row_parallel_forward_local(const void* X, int x_dtype, int64_t ldx, const void* W,
                                                     int w_dtype, int64_t ldw, float* Y, int64_t ldy, int64_t M,
                                                     int64_t N, int64_t K, int tp, void* stream) {
  TBIK_TRY(check_dense(X, x_dtype, M, K, ldx, "X"));
  TBIK_TRY(check_dense(W, w_dtype, K, N, ldw, "W"));
  TBIK_TRY(check_dense(Y, TBIK_F32, M, N, ldy, "Y"));
  if (tp < 1 || (tp & (tp - 1)) || tp > kMaxRanks) return set_error(TBIK_BAD_WORLD_SIZE, "tp must be a power of two");
  if (K % tp)  // layers.cpp:106-111
    return set_error(TBIK_SHARD_ERROR, "baseline row shard: K=" + std::to_string(K) + " not divisible by tp=" +
                                           std::to_string(tp));
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t width = K / tp;
  const size_t slice = static_cast<size_t>(M) * N;
  float* parts = static_cast<float*>(workspace(slice * tp * sizeof(float), 11, s));
  if (!parts) return set_error(TBIK_CUDA_ERROR, "workspace allocation failed");
  PartPtrs pp{};
  for (int r = 0; r < tp; ++r) {
    const char* Xr = static_cast<const char*>(X) + r * width * esize(x_dtype);
    const char* Wr = static_cast<const char*>(W) + r * width * ldw * esize(w_dtype);
    TBIK_TRY(blas_gemm(Xr, x_dtype, ldx, Wr, w_dtype, ldw, parts + slice * r, TBIK_F32, N, M, N, width, s));
    pp.p[r] = parts + slice * r;
  }
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((static_cast<int64_t>(slice) + 255) / 256, 148 * 4));
  ring_sum_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(pp, tp, M, N, Y, ldy);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_baseline_column_parallel_forward_local(const void* X, int x_dtype, int64_t ldx, const void* W,
                                                        int w_dtype, int64_t ldw, float* Y, int64_t ldy, int64_t M,
                                                        int64_t N, int64_t K, int tp, void* stream) {
  TBIK_TRY(check_dense(X, x_dtype, M, K, ldx, "X"));
  TBIK_TRY(check_dense(W, w_dtype, K, N, ldw, "W"));
  TBIK_TRY(check_dense(Y, TBIK_F32, M, N, ldy, "Y"));
  int64_t bounds[2 * kMaxRanks];
  if (tp < 1 || tp > kMaxRanks) return set_error(TBIK_BAD_WORLD_SIZE, "tp out of range");
  TBIK_TRY(tbik_make_column_shard_plan(N, tp, bounds));
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int r = 0; r < tp; ++r) {
    const int64_t b = bounds[2 * r], e = bounds[2 * r + 1];
    TBIK_TRY(blas_gemm(X, x_dtype, ldx, static_cast<const char*>(W) + b * esize(w_dtype), w_dtype, ldw, Y + b,
                       TBIK_F32, ldy, M, e - b, K, s));
  }
  return TBIK_OK;
}

static_assert(sizeof(ncclUniqueId) <= TBIK_NCCL_ID_BYTES, "nccl id size");

tbik_status tbik_nccl_unique_id(void* id_out) {
  if (!id_out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_error(TBIK_CUDA_ERROR, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  std::memset(id_out, 0, TBIK_NCCL_ID_BYTES);
  std::memcpy(id_out, &id, sizeof(id));
  return TBIK_OK;
}

tbik_status tbik_nccl_comm_create(int world_size, int rank, int device, const void* id, void** comm) {
  if (!id || !comm) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  TBIK_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = ncclCommInitRank(&c, world_size, uid, rank);
  if (r != ncclSuccess) return set_error(TBIK_CUDA_ERROR, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  *comm = c;
  return TBIK_OK;
}

tbik_status tbik_nccl_comm_destroy(void* comm) {
  if (comm) ncclCommDestroy(static_cast<ncclComm_t>(comm));
  return TBIK_OK;
}

tbik_status tbik_baseline_cublas_nccl(void* comm, const void* X_shard, int x_dtype, int64_t ldx, const void* W_shard,
                                      int w_dtype, int64_t ldw, void* Y, int64_t M, int64_t N, int64_t K_shard,
                                      int out_f32, void* stream) {
  if (!comm || !Y) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  TBIK_TRY(check_dense(X_shard, x_dtype, M, K_shard, ldx, "X"));
  TBIK_TRY(check_dense(W_shard, w_dtype, K_shard, N, ldw, "W"));
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int cdt = out_f32 ? TBIK_F32 : TBIK_BF16;
  TBIK_TRY(blas_gemm(X_shard, x_dtype, ldx, W_shard, w_dtype, ldw, Y, cdt, N, M, N, K_shard, s));
  const ncclResult_t r = ncclAllReduce(Y, Y, static_cast<size_t>(M) * N, out_f32 ? ncclFloat32 : ncclBfloat16, ncclSum,
                                       static_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) return set_error(TBIK_CUDA_ERROR, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  return TBIK_OK;
}

}  // extern "C"
