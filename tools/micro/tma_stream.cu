// tma_stream.cu -- how fast can TMA stream a 14336 x 4096 bf16 weight matrix into
// shared memory on B200, as a function of the CTA's strip shape?  (Decode-regime
// calibration for tbik_gemm_skinny.cu; the consumer only releases the stage.)
//   ./tma_stream  -> one line per variant: us per full pass, GB/s
// Variants: strip width (columns per CTA, in 64-column SW128 boxes), K units
// (CTAs along K), box rows, stages.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol) : "memory");
}

struct P { int K, N, strip_boxes, units, box_rows, stages, hint, xrows; };

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tx, const P p) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = p.strip_boxes * p.box_rows * 128 + p.xrows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int strips = p.N / (64 * p.strip_boxes);
  const int strip = blockIdx.x % strips, unit = blockIdx.x / strips;
  const int krows = p.K / p.units;
  const int k0 = unit * krows;
  const int nst = krows / p.box_rows;
  uint64_t pol;
  if (p.hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  if (warp == 0 && lane == 0) {
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < nst; ++i) {
      mbar_wait(&empty[st], ph ^ 1);
      mbar_arrive_expect_tx(&full[st], stage_bytes);
      for (int b = 0; b < p.strip_boxes; ++b)
        tma_load_2d(sm + st * stage_bytes + b * p.box_rows * 128, &tm, &full[st], (strip * p.strip_boxes + b) * 64, k0 + i * p.box_rows, pol);
      if (p.xrows) tma_load_2d(sm + st * stage_bytes + p.strip_boxes * p.box_rows * 128, &tx, &full[st], k0 + i * p.box_rows, 0, pol);
      if (++st == p.stages) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < nst; ++i) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == p.stages) { st = 0; ph ^= 1; }
    }
  }
  __syncthreads();
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int K = 14336, N = 4096;
  const size_t bytes = size_t(K) * N * 2;
  std::vector<void*> bufs(4);
  for (auto& b : bufs) { CK(cudaMalloc(&b, bytes)); CK(cudaMemset(b, 1, bytes)); }
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncFn enc = reinterpret_cast<EncFn>(fn);
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 230000));
  struct V { int strip_boxes, units, box_rows, stages, hint, promo, xrows; };
  std::vector<V> vs = {
      {2, 4, 64, 11, 0, 2, 0}, {2, 4, 64, 11, 0, 2, 16}, {2, 4, 64, 9, 0, 2, 64}, {2, 4, 64, 7, 0, 2, 128},
      {2, 4, 64, 7, 0, 2, 0}, {2, 4, 64, 4, 0, 2, 0}, {2, 4, 64, 7, 1, 2, 128},
  };
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  void* xbuf; CK(cudaMalloc(&xbuf, size_t(128) * K * 2)); CK(cudaMemset(xbuf, 0, size_t(128) * K * 2));
  for (const V& v : vs) {
    std::vector<CUtensorMap> maps(4);
    CUtensorMap xm;
    if (v.xrows) {
      cuuint64_t dims[2] = {cuuint64_t(K), 128}; cuuint64_t str[1] = {cuuint64_t(K) * 2};
      cuuint32_t box[2] = {64, cuuint32_t(v.xrows)}; cuuint32_t es[2] = {1, 1};
      if (enc(&xm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xbuf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) return 1;
    } else xm = maps[0];
    for (int i = 0; i < 4; ++i) {
      cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(K)}; cuuint64_t str[1] = {cuuint64_t(N) * 2};
      cuuint32_t box[2] = {64, cuuint32_t(v.box_rows)}; cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, bufs[i], dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, v.promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : v.promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return 1; }
    }
    P p{K, N, v.strip_boxes, v.units, v.box_rows, v.stages, v.hint, v.xrows};
    if (!v.xrows) xm = maps[0];
    const int strips = N / (64 * v.strip_boxes);
    const int grid = strips * v.units;
    const size_t smem = 1024 + size_t(v.stages) * (v.strip_boxes * v.box_rows * 128 + v.xrows * 128) + 1024;
    if (smem > 230000) { printf("skip smem\n"); continue; }
    for (int i = 0; i < 4; ++i) stream_kernel<<<grid, 64, smem>>>(maps[i], xm, p);
    CK(cudaDeviceSynchronize());
    const int reps = 40;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) stream_kernel<<<grid, 64, smem>>>(maps[i % 4], xm, p);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("strip %4d cols  units %3d  grid %4d  box_rows %3d  stages %2d  stage %6d B  hint %d promo %d xrows %3d : %6.1f us  %6.0f GB/s\n",
           v.strip_boxes * 64, v.units, grid, v.box_rows, v.stages, v.strip_boxes * v.box_rows * 128, v.hint, v.promo, v.xrows, us, bytes / us / 1e3);
  }
  return 0;
}
