// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM with 4 / 8 / 16 warps,
// and the cost of ld + 32 FADD per chunk (the TBIK merge inner step).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2511_17826_b200/csrc/tbik_common.cuh"
using namespace tbik_b200;

template <int MODE>
__global__ void k(unsigned long long* out, int iters, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
  float acc[32];
  for (int i = 0; i < 32; ++i) acc[i] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float v[32];
    tmem_ld32(base + ((it & 3) * 128) % 512, v);
    if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = __fadd_rn(acc[i], v[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = __uint_as_float(__float_as_uint(acc[i]) ^ __float_as_uint(v[i]));
    }
  }
  long long t1 = clock64();
  __syncthreads();
  float s = 0;
  for (int i = 0; i < 32; ++i) s += acc[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}

int main() {
  unsigned long long* d; float* sink;
  cudaMalloc(&d, 8 * 148); cudaMalloc(&sink, 4 * 148 * 512);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16}) {
      if (mode == 0) k<0><<<148, warps * 32>>>(d, iters, sink); else k<1><<<148, warps * 32>>>(d, iters, sink);
      cudaDeviceSynchronize();
      if (mode == 0) k<0><<<148, warps * 32>>>(d, iters, sink); else k<1><<<148, warps * 32>>>(d, iters, sink);
      cudaDeviceSynchronize();
      unsigned long long h[148]; cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
      double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
      double bytes = (double)iters * warps * 32 * 32 * 4;
      printf("%s warps=%2d: %.1f cycles per warp-ld, %.1f B/clk/SM TMEM read\n",
             mode ? "ld+32FADD" : "ld only  ", warps, cyc / iters, bytes / cyc);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
