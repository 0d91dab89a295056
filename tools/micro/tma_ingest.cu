// tma_ingest.cu -- per-SM TMA ingest of a decode-sized TP shard (K = 1792 rows x
// N = 4096 bf16 = 14.7 MB, L2-resident after the first pass): each CTA streams one
// column strip of the matrix through an NST-stage ring of {cols x 64 rows} boxes.
//   strip 64 cols, 128B swizzle -> 64 CTAs x 229 KB   (the skinny kernel's TP = 8 shard)
//   strip 32 cols,  64B swizzle -> 128 CTAs x 115 KB  (half the bytes per CTA, 64-byte rows)
//   strip 128 cols as 2 x 64    -> 32 CTAs x 458 KB
// Question: is a CTA's ingest bound by bytes or by TMA row requests?
// Finding (profiles/r02_tma_ingest.txt): ~520-600 cycles per ring stage whatever
// its bytes (4-32 KB), box count or in-flight depth -- a property of this one-
// thread wait-then-reissue loop, not of TMA: the skinny kernel streams the same
// strips twice as fast (its bound is the MMA count, tools/micro/small_mma.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_ingest tma_ingest.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 3D mode (transposed == 2): one box {64 cols, rows, cols / 64} covers the strip's
// 64-column slabs of `rows` rows in one TMA instruction.
// X mode (transposed == 3): the strip is a token block X[M = cols][K] streamed in
// K: {64 K, M rows} boxes (boxes_per_stage of them per stage), or (transposed == 4)
// one 3D box {64 K, M rows, boxes_per_stage} per stage.
// One thread streams the strip: keeps NST box loads in flight, consumes in order.
__global__ void ingest(const __grid_constant__ CUtensorMap tm, int K, int cols, int boxes_per_stage, int nst,
                       int rows, int transposed, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int box_bytes = (cols / boxes_per_stage) * rows * 2;
  const int stage_bytes = box_bytes * boxes_per_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + nst * stage_bytes);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long long t0 = clock64();
  const int n0 = blockIdx.x * cols, nk = K / rows;
  int issued = 0;
  for (; issued < nst && issued < nk; ++issued) {
    mbar_expect(&full[issued], stage_bytes);
    for (int b = 0; b < boxes_per_stage; ++b)
      if (transposed == 2) {
        if (b == 0) tma3d(sm + issued * stage_bytes, &tm, &full[issued], 0, issued * rows, n0 / 64);
      } else if (transposed == 1)  // [N][K]: inner = K (rows of the strip's box), outer = N
        tma2d(sm + issued * stage_bytes + b * box_bytes, &tm, &full[issued], issued * rows, n0 + b * (cols / boxes_per_stage));
      else
        tma2d(sm + issued * stage_bytes + b * box_bytes, &tm, &full[issued], n0 + b * (cols / boxes_per_stage), issued * rows);
  }
  for (int k = 0; k < nk; ++k) {
    const int s = k % nst;
    mbar_wait(&full[s], (k / nst) & 1);
    if (issued < nk) {
      const int si = issued % nst;
      mbar_expect(&full[si], stage_bytes);
      for (int b = 0; b < boxes_per_stage; ++b)
        if (transposed == 2) {
          if (b == 0) tma3d(sm + si * stage_bytes, &tm, &full[si], 0, issued * rows, n0 / 64);
        } else if (transposed == 1)
          tma2d(sm + si * stage_bytes + b * box_bytes, &tm, &full[si], issued * rows, n0 + b * (cols / boxes_per_stage));
        else
          tma2d(sm + si * stage_bytes + b * box_bytes, &tm, &full[si], n0 + b * (cols / boxes_per_stage), issued * rows);
      ++issued;
    }
  }
  cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int K = 1792, N = 4096;
  void* buf;
  cudaMalloc(&buf, size_t(K) * N * 2);
  cudaMemset(buf, 1, size_t(K) * N * 2);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncFn enc = reinterpret_cast<EncFn>(fn);
  EncFn enc3 = enc;
  unsigned long long* dc;
  cudaMalloc(&dc, 8 * 512);
  cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  struct V { int cols, boxes, nst, rows, tr; CUtensorMapSwizzle sw; const char* name; };
  std::vector<V> vs = {{64, 1, 16, 64, 0, CU_TENSOR_MAP_SWIZZLE_128B, "[K][N] 64-col strips, 64-row boxes"},
                       {32, 1, 16, 64, 0, CU_TENSOR_MAP_SWIZZLE_64B, "[K][N] 32-col strips, 64B rows"},
                       {128, 2, 8, 64, 0, CU_TENSOR_MAP_SWIZZLE_128B, "[K][N] 128-col strips (2 x 64)"},
                       {64, 1, 16, 32, 0, CU_TENSOR_MAP_SWIZZLE_128B, "[K][N] 64-col strips, 32-row boxes"},
                       {64, 1, 8, 128, 0, CU_TENSOR_MAP_SWIZZLE_128B, "[K][N] 64-col strips, 128-row boxes"},
                       {64, 1, 16, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B, "[N][K] 64-row strips, 64-K boxes"},
                       {32, 1, 16, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B, "[N][K] 32-row strips, 64-K boxes"},
                       // in-flight depth: latency- or service-bound?
                       {64, 1, 4, 64, 0, CU_TENSOR_MAP_SWIZZLE_128B, "64-row boxes, NST 4"},
                       {64, 1, 8, 64, 0, CU_TENSOR_MAP_SWIZZLE_128B, "64-row boxes, NST 8"},
                       {64, 1, 24, 64, 0, CU_TENSOR_MAP_SWIZZLE_128B, "64-row boxes, NST 24"},
                       {64, 1, 8, 32, 0, CU_TENSOR_MAP_SWIZZLE_128B, "32-row boxes, NST 8"},
                       {64, 1, 32, 32, 0, CU_TENSOR_MAP_SWIZZLE_128B, "32-row boxes, NST 32"},
                       {64, 1, 48, 32, 0, CU_TENSOR_MAP_SWIZZLE_128B, "32-row boxes, NST 48"},
                       {64, 1, 4, 128, 0, CU_TENSOR_MAP_SWIZZLE_128B, "128-row boxes, NST 4"},
                       {64, 1, 12, 128, 0, CU_TENSOR_MAP_SWIZZLE_128B, "128-row boxes, NST 12"},
                       {64, 1, 4, 256, 0, CU_TENSOR_MAP_SWIZZLE_128B, "256-row boxes, NST 4"},
                       {64, 1, 6, 256, 0, CU_TENSOR_MAP_SWIZZLE_128B, "256-row boxes, NST 6"},
                       {32, 1, 8, 256, 0, CU_TENSOR_MAP_SWIZZLE_64B, "32-col strips, 256-row boxes, NST 8"},
                       {32, 1, 7, 256, 0, CU_TENSOR_MAP_SWIZZLE_64B, "32-col strips, 256-row boxes, NST 7"},
                       {128, 2, 8, 64, 2, CU_TENSOR_MAP_SWIZZLE_128B, "128-col strips, one 3D box {64,64,2}"},
                       {128, 2, 4, 128, 2, CU_TENSOR_MAP_SWIZZLE_128B, "128-col strips, one 3D box {64,128,2}"},
                       {256, 4, 4, 64, 2, CU_TENSOR_MAP_SWIZZLE_128B, "256-col strips, one 3D box {64,64,4}"}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const V& v : vs) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(K)}, str[1] = {cuuint64_t(N) * 2};
    cuuint32_t box[2] = {cuuint32_t(v.cols / v.boxes), cuuint32_t(v.rows)}, es[2] = {1, 1};
    if (v.tr == 2) {  // {64 cols, K rows, N / 64 slabs}: slab stride 128 B
      cuuint64_t d3[3] = {64, cuuint64_t(K), cuuint64_t(N / 64)}, s3[2] = {cuuint64_t(N) * 2, 128};
      cuuint32_t b3[3] = {64, cuuint32_t(v.rows), cuuint32_t(v.boxes)}, e3[3] = {1, 1, 1};
      if (enc3(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode3 failed\n");
        return 1;
      }
    } else if (v.tr) {  // the same bytes viewed as W^T: [N][K], K contiguous
      dims[0] = K; dims[1] = N; str[0] = cuuint64_t(K) * 2;
      box[0] = cuuint32_t(v.rows); box[1] = cuuint32_t(v.cols / v.boxes);
    }
    if (v.tr != 2 && enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    const int grid = N / v.cols;
    const size_t smem = 1024 + size_t(v.nst) * v.cols * v.rows * 2 + 1024;
    for (int r = 0; r < 3; ++r) ingest<<<grid, 32, smem>>>(m, K, v.cols, v.boxes, v.nst, v.rows, v.tr, dc);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) ingest<<<grid, 32, smem>>>(m, K, v.cols, v.boxes, v.nst, v.rows, v.tr, dc);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(grid);
    cudaMemcpy(h.data(), dc, 8 * grid, cudaMemcpyDeviceToHost);
    double c = 0;
    for (auto x : h) c += x;
    c /= grid;
    const double per_cta = double(K) * v.cols * 2;
    printf("%-38s grid %3d: %6.2f us/pass, %7.0f cycles per CTA = %5.1f B/clk per SM, total %6.0f GB/s (%s)\n", v.name,
           grid, ms * 1e3 / 20, c, per_cta / c, double(K) * N * 2 / (ms * 1e-3 / 20) / 1e9, cudaGetErrorString(e));
  }
  return 0;
}
