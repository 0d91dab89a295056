// small_mma.cu -- cost of one tcgen05.mma (cta_group::1, kind::f16, K = 16) with the
// skinny (decode) kernel's operand shapes: A = a weight slice (M = 64 / 128 rows,
// MN-major as the [K][N] weight is stored, or K-major), B = the tokens (N = 16 ..
// 256, K-major).  Operands stay resident in shared memory (no TMA); one thread
// issues R MMAs into one accumulator (a dependent chain, like one leaf) or rotating
// over 4 accumulators (independent chains), then commits and waits.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../include -o small_mma small_mma.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../../paper_2511_17826_b200/csrc/tbik_common.cuh"

using namespace tbik_b200;

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

// a_mn: A MN-major (SW128, 64-row atoms 8 KB apart, K groups of 8 rows 1 KB apart,
// +2 KB per K = 16) or K-major (SW128 128-byte rows, +32 B per K = 16, 8-row
// groups 1 KB apart).  B K-major SW128.  nacc accumulators of N columns.
__global__ void k_small(int M, int N, int a_mn, int nacc, int reps, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;           // 64 KB region (A: 128 x 64 K at most = 16 KB per 64 K)
  uint8_t* sB = smem + 65536;   // 64 KB region
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 131072);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *slot;
  if (warp == 0) {  // warp-uniform loop, one elected lane issues (the kernels' pattern)
    const uint32_t idesc = umma_idesc_bf16(M, N, a_mn, 0);
    const uint64_t ad0 = a_mn ? desc(smem_u32(sA), 8192, 1024, 2) : desc(smem_u32(sA), 16, 1024, 2);
    const uint64_t bd0 = desc(smem_u32(sB), 16, 1024, 2);
    const uint64_t astep = a_mn ? (2048 >> 4) : (32 >> 4), bstep = 32 >> 4;
    const long long t0 = clock64();
    for (int r = 0; r < reps; r += 16) {
      const uint32_t d = tbase + static_cast<uint32_t>(((r >> 4) % nacc) * N);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          umma_bf16(d, ad0 + (kk & 3) * astep, bd0 + (kk & 3) * bstep, idesc, (r >= 16 * nacc || kk) ? 1u : 0u);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(bar);
    __syncwarp();
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = static_cast<unsigned long long>(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int smem = 131072 + 2048;
  cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct V { int M, N, a_mn, nacc; };
  const V vs[] = {{128, 16, 1, 1}, {128, 16, 0, 1}, {128, 16, 1, 4}, {128, 16, 0, 4}, {64, 16, 1, 1},
                  {64, 16, 0, 1},  {128, 32, 1, 1}, {128, 64, 1, 1}, {128, 128, 1, 1}, {128, 256, 1, 1},
                  {128, 64, 0, 1}, {128, 128, 0, 1}, {128, 256, 0, 1}, {128, 32, 1, 4}, {64, 64, 1, 1},
                  {128, 8, 1, 1}, {64, 8, 1, 1}, {128, 192, 1, 1}};
  const int reps = 1024;
  for (const V& v : vs) {
    unsigned long long best = ~0ull;
    for (int t = 0; t < 5; ++t) {
      k_small<<<1, 128, smem>>>(v.M, v.N, v.a_mn, v.nacc, reps, d);
      unsigned long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      if (h < best) best = h;
    }
    const double floor_ = (v.M < 128 ? 128 : v.M) * v.N / 256.0;
    printf("M %3d N %3d A %s acc %d: %6.1f cycles per MMA (floor %5.1f) %s\n", v.M, v.N, v.a_mn ? "MN-major" : "K-major ",
           v.nacc, double(best) / reps, floor_, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
