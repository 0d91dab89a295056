// tbik_hostio.cu -- the reference's Matrix-in / Matrix-out calls with HOST
// buffers (tree_matmul, matmul.hpp:53; row_parallel_forward, layers.hpp:43-45):
// the activations arrive from host memory and the f32 result goes back to it,
// while the weights stay resident in HBM.
//
// The copies are pipelined with the tensor cores over row chunks:
//
//   h2d stream   A[c0] -> dA[0]   A[c1] -> dA[1]   A[c2] -> dA[0] ...
//   `stream`               GEMM c0          GEMM c1          GEMM c2 ...
//   d2h stream                      dC[0] -> C[c0]   dC[1] -> C[c1] ...
//
// so PCIe runs in both directions at once and the GEMM hides under the
// transfers.  Splitting the rows is invisible in the bits: every output row is
// the same function of its own A row at any M (batch invariance; the per-element
// tree never depends on M).  Double-buffered staging in the caller stream's arena
// (slots 4-7); cross-stream order through events only, so the call returns as
// soon as the work is enqueued and `stream` is ordered after the last D2H.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "tbik_common.cuh"
#include "tbik_internal.h"

namespace tbik_b200 {

namespace {

struct HostIoCtx {
  bool init = false;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t start, h2d_done[2], comp_done[2], d2h_done[2];
};
std::mutex g_hio_mu;
// One copy-stream pair + events per (device, caller stream): two callers on two
// streams never share staging buffers (workspace is keyed the same way) or events.
std::map<std::pair<int, uintptr_t>, HostIoCtx> g_hio;

tbik_status ctx_for_stream(cudaStream_t s, HostIoCtx** out) {
  int dev = 0;
  TBIK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_hio_mu);
  HostIoCtx& c = g_hio[{dev, reinterpret_cast<uintptr_t>(s)}];
  if (!c.init) {
    TBIK_CUDA(cudaStreamCreateWithFlags(&c.h2d, cudaStreamNonBlocking));
    TBIK_CUDA(cudaStreamCreateWithFlags(&c.d2h, cudaStreamNonBlocking));
    TBIK_CUDA(cudaEventCreateWithFlags(&c.start, cudaEventDisableTiming));
    for (int b = 0; b < 2; ++b) {
      TBIK_CUDA(cudaEventCreateWithFlags(&c.h2d_done[b], cudaEventDisableTiming));
      TBIK_CUDA(cudaEventCreateWithFlags(&c.comp_done[b], cudaEventDisableTiming));
      TBIK_CUDA(cudaEventCreateWithFlags(&c.d2h_done[b], cudaEventDisableTiming));
    }
    c.init = true;
  }
  *out = &c;
  return TBIK_OK;
}

size_t esize(int dt) { return dt == TBIK_BF16 ? 2 : 4; }

int64_t default_chunk(int64_t M) {
  // ~8 chunks (pipeline fill = one chunk each way), never below 256 rows so each
  // chunk's GEMM still fills the machine with 256-row pair tiles.
  int64_t c = (M + 7) / 8;
  c = (c + 127) / 128 * 128;
  return std::max<int64_t>(c, 256);
}

// compute(dA, lda_dev, dC, ldc_dev, rows, stream)
template <class F>
tbik_status pipeline(const void* A_host, int adt, int64_t lda, int64_t K, float* C_host, int64_t ldc, int64_t M,
                     int64_t N, int64_t chunk, cudaStream_t s, F compute) {
  HostIoCtx* cx = nullptr;
  TBIK_TRY(ctx_for_stream(s, &cx));
  // Row chunks: a fixed size when the caller asks for one; by default ramped
  // (128, 256, then up to 512, then 256, 128) so the pipeline fills and drains on
  // small copies while the bulk moves in large ones.
  std::vector<int64_t> sizes;
  if (chunk > 0) {
    chunk = std::min(chunk, M);
    for (int64_t r = 0; r < M; r += chunk) sizes.push_back(std::min(chunk, M - r));
  } else if (M >= 1024) {
    chunk = default_chunk(M);
    const int64_t mid = M - 768;
    sizes = {128, 256};
    for (int64_t r = 0; r < mid; r += chunk) sizes.push_back(std::min(chunk, mid - r));
    sizes.push_back(256);
    sizes.push_back(128);
  } else {
    chunk = std::min(default_chunk(M), M);
    for (int64_t r = 0; r < M; r += chunk) sizes.push_back(std::min(chunk, M - r));
  }
  const size_t es = esize(adt);
  const size_t a_bytes = static_cast<size_t>(chunk) * K * es, c_bytes = static_cast<size_t>(chunk) * N * 4;
  char* dA[2];
  float* dC[2];
  for (int b = 0; b < 2; ++b) {
    dA[b] = static_cast<char*>(workspace(a_bytes, 4 + b, s));
    dC[b] = static_cast<float*>(workspace(c_bytes, 6 + b, s));
    if (!dA[b] || !dC[b]) return set_error(TBIK_CUDA_ERROR, "host-io staging allocation failed");
  }
  TBIK_CUDA(cudaEventRecord(cx->start, s));
  TBIK_CUDA(cudaStreamWaitEvent(cx->h2d, cx->start, 0));
  const int64_t nchunks = static_cast<int64_t>(sizes.size());
  int64_t r0 = 0;
  for (int64_t i = 0; i < nchunks; r0 += sizes[i], ++i) {
    const int b = static_cast<int>(i & 1);
    const int64_t rows = sizes[i];
    if (i >= 2) TBIK_CUDA(cudaStreamWaitEvent(cx->h2d, cx->comp_done[b], 0));  // dA[b] consumed
    if (lda == K)  // contiguous rows: one linear copy (the 2D path is slower on the copy engines)
      TBIK_CUDA(cudaMemcpyAsync(dA[b], static_cast<const char*>(A_host) + r0 * lda * es, rows * K * es,
                                cudaMemcpyHostToDevice, cx->h2d));
    else
      TBIK_CUDA(cudaMemcpy2DAsync(dA[b], K * es, static_cast<const char*>(A_host) + r0 * lda * es, lda * es,
                                  K * es, rows, cudaMemcpyHostToDevice, cx->h2d));
    TBIK_CUDA(cudaEventRecord(cx->h2d_done[b], cx->h2d));
    TBIK_CUDA(cudaStreamWaitEvent(s, cx->h2d_done[b], 0));
    if (i >= 2) TBIK_CUDA(cudaStreamWaitEvent(s, cx->d2h_done[b], 0));  // dC[b] drained
    TBIK_TRY(compute(dA[b], K, dC[b], N, rows, s));
    TBIK_CUDA(cudaEventRecord(cx->comp_done[b], s));
    TBIK_CUDA(cudaStreamWaitEvent(cx->d2h, cx->comp_done[b], 0));
    if (ldc == N)
      TBIK_CUDA(cudaMemcpyAsync(C_host + r0 * ldc, dC[b], rows * N * sizeof(float), cudaMemcpyDeviceToHost, cx->d2h));
    else
      TBIK_CUDA(cudaMemcpy2DAsync(C_host + r0 * ldc, ldc * sizeof(float), dC[b], N * sizeof(float),
                                  N * sizeof(float), rows, cudaMemcpyDeviceToHost, cx->d2h));
    TBIK_CUDA(cudaEventRecord(cx->d2h_done[b], cx->d2h));
  }
  TBIK_CUDA(cudaStreamWaitEvent(s, cx->d2h_done[(nchunks - 1) & 1], 0));
  return TBIK_OK;
}

tbik_status check_host_args(const void* A, int adt, int64_t lda, const void* B, int bdt, int64_t ldb, const float* C,
                            int64_t ldc, int64_t M, int64_t N, int64_t K) {
  if (M < 1 || N < 1 || K < 1) return set_error(TBIK_BAD_DIMENSION, "dimensions must be >= 1");
  if ((adt != TBIK_F32 && adt != TBIK_BF16) || (bdt != TBIK_F32 && bdt != TBIK_BF16))
    return set_error(TBIK_UNKNOWN_DTYPE, "dtype");
  if (!A || !B || !C) return set_error(TBIK_BAD_ARGUMENT, "null pointer");
  if (lda < K || ldb < N || ldc < N) return set_error(TBIK_BAD_ARGUMENT, "leading dimension < cols");
  return TBIK_OK;
}

}  // namespace
}  // namespace tbik_b200

using namespace tbik_b200;

extern "C" {

tbik_status tbik_tree_matmul_hostio(const void* A_host, int a_dtype, int64_t lda, const void* B, int b_dtype,
                                    int64_t ldb, float* C_host, int64_t ldc, int64_t M, int64_t N, int64_t K,
                                    const tbik_block_config* cfg, int leaf_mode, int64_t chunk_rows, void* stream) {
  if (!cfg) return set_error(TBIK_BAD_ARGUMENT, "null cfg");
  TBIK_TRY(check_host_args(A_host, a_dtype, lda, B, b_dtype, ldb, C_host, ldc, M, N, K));
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 CUDA device (no CPU fallback)");
  return pipeline(A_host, a_dtype, lda, K, C_host, ldc, M, N, chunk_rows, static_cast<cudaStream_t>(stream),
                  [&](const void* dA, int64_t ldad, float* dC, int64_t ldcd, int64_t rows, cudaStream_t s) {
                    return tbik_tree_matmul(dA, a_dtype, ldad, B, b_dtype, ldb, dC, ldcd, rows, N, K, cfg,
                                            leaf_mode, s);
                  });
}

tbik_status tbik_group_row_parallel_forward_hostio(tbik_group* g, const void* X_host_shard, int x_dtype,
                                                   int64_t ldx, const void* W_shard, int w_dtype, int64_t ldw,
                                                   float* Y_host, int64_t ldy, int64_t M, int64_t N, int64_t K_shard,
                                                   int64_t K_global, const tbik_block_config* cfg, int64_t c_max,
                                                   int leaf_mode, int64_t chunk_rows, void* stream) {
  if (!g || !cfg) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  TBIK_TRY(check_host_args(X_host_shard, x_dtype, ldx, W_shard, w_dtype, ldw, Y_host, ldy, M, N, K_shard));
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 CUDA device (no CPU fallback)");
  int64_t bounds[2 * kMaxRanks];
  TBIK_TRY(tbik_make_row_shard_plan(K_global, cfg, tbik_group_world_size(g), c_max, bounds));
  const int r = tbik_group_rank(g);
  if (bounds[2 * r + 1] - bounds[2 * r] != K_shard)
    return set_error(TBIK_SHAPE_MISMATCH, "X shard width does not match this rank's make_row_shard_plan range");
  // Every rank must cut the same chunks (one collective epoch per chunk): the
  // chunking depends only on (M, chunk_rows), which all ranks share.
  return pipeline(X_host_shard, x_dtype, ldx, K_shard, Y_host, ldy, M, N, chunk_rows, static_cast<cudaStream_t>(stream),
                  [&](const void* dX, int64_t ldxd, float* dY, int64_t ldyd, int64_t rows, cudaStream_t s) {
                    return tbik_group_row_parallel_forward(g, dX, x_dtype, ldxd, W_shard, w_dtype, ldw, dY, ldyd,
                                                           rows, N, K_global, cfg, c_max, leaf_mode, s);
                  });
}

}  // extern "C"
