// Feasibility check: tcgen05.mma.cta_group::2 with A read from TMEM (TS form), A
// staged SMEM -> TMEM by tcgen05.cp.cta_group::2.128x256b from the TMA's 128B-swizzled
// K-major tile, against the SS form (A from shared memory) on the same data.
//   D[256 x N] = A[256 x K] . B[K x N], K = 64 (4 K=16 steps), one CTA pair.
// B is MN-major: N = 128 -> each CTA stages 64 columns as one SW128 atom; N = 96 ->
// 48 columns as three SW32 atoms (16 columns each).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o ts_mma ts_mma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../paper_2511_17826_b200/csrc/tbik_common.cuh"
#include "../../paper_2511_17826_b200/csrc/tbik_pair.cuh"

using namespace tbik_b200;
using namespace tbik_b200::pair_ptx;

constexpr int K = 64;

__device__ __forceinline__ void umma_ts_2cta(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void utccp_2cta(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

// mode 0: SS, mode 1: TS (A via tcgen05.cp)
template <int N>
__global__ void __cluster_dims__(2, 1, 1) k_pair(const __grid_constant__ CUtensorMap tmA,
                                                  const __grid_constant__ CUtensorMap tmB, float* out, int mode) {
  constexpr int NC = N / 2;  // B columns per CTA
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;          // 16 KB: 128 rows x 64 K, SW128
  uint8_t* sB = smem + 16384;  // NC cols x 64 K
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 32768);
  uint64_t* done = full + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_rank() & 1;
  if (threadIdx.x == 0) {
    mbar_init(full, 2);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_2cta(tslot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t fb = mapa(smem_u32(full), 0);
    const uint32_t tx = 16384 + NC * K * 2;
    if (rank == 0)
      mbar_arrive_expect_tx(full, tx);
    else
      mbar_arrive_expect_tx_cluster(fb, tx);
    tma_load_2d_2sm(sA, &tmA, fb, 0, rank * 128);
    if (N == 128) {
      tma_load_2d_2sm(sB, &tmB, fb, rank * 64, 0);
    } else {
      for (int a = 0; a < NC / 16; ++a) tma_load_2d_2sm(sB + a * 16 * K * 2, &tmB, fb, rank * NC + a * 16, 0);
    }
  }
  if (rank == 0 && warp == 1) {
    mbar_wait(full, 0);
    tc_fence_after();
    if (elect_one()) {
      constexpr uint32_t IDESC = umma_idesc_bf16(256, N, 0, 1);
      const uint32_t d = tbase;            // cols [0, N)
      const uint32_t ta = tbase + 256;     // A in TMEM: 4 K-steps x 8 columns
      if (mode == 1) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) utccp_2cta(ta + kk * 8, desc(smem_u32(sA) + kk * 32, 16, 1024, 2));
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t bdesc;
        if (N == 128)
          bdesc = desc(smem_u32(sB) + kk * 2048, 8192, 1024, 2);  // SW128 MN-major
        else
          bdesc = desc(smem_u32(sB) + kk * 512, 16 * K * 2, 256, 6);  // SW32 MN-major: atoms 2 KB apart
        if (mode == 1)
          umma_ts_2cta(d, ta + kk * 8, bdesc, IDESC, kk != 0);
        else
          umma_bf16_2cta(d, desc(smem_u32(sA) + kk * 32, 16, 1024, 2), bdesc, IDESC, kk != 0);
      }
      umma_commit_2cta(done, 0x3);
    }
    __syncwarp();
  }
  mbar_wait(done, 0);
  tc_fence_after();
  // drain: 4 warps, lane quarter = warp, rows rank*128 + 32 warp + lane
  const int row = rank * 128 + warp * 32 + (threadIdx.x & 31);
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tmem_ld32(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
    for (int i = 0; i < 32 && c + i < N; ++i) out[row * N + c + i] = v[i];
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc_2cta(tbase, 512);
}

// Throughput: per "leaf" (K = 256 = 4 x 64): mode 0 = 16 SS MMAs at N=192 (one tile),
// mode 1 = 2 halves x 16 TS MMAs at N=96 + 16 tcgen05.cp (A for the next leaf),
// mode 2 = 2 halves x 16 SS MMAs at N=96 (A read twice), mode 3 = 16 SS N=128 (the
// 256x128 kernel's per-leaf work, for scale).  Operands stay resident in smem.
__global__ void __cluster_dims__(2, 1, 1) k_tput(int leaves, int mode, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;            // 4 stages x 16 KB (garbage data is fine)
  uint8_t* sB = smem + 65536;    // 4 stages x 2 halves x 6 KB (SW32)
  uint64_t* done = reinterpret_cast<uint64_t*>(smem + 65536 + 49152);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_rank() & 1;
  if (threadIdx.x == 0) {
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_2cta(tslot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (rank == 0 && warp == 1 && elect_one()) {
    const long long t0 = clock64();
    for (int l = 0; l < leaves; ++l) {
      if (mode == 0 || mode == 3) {
        const int n = mode == 0 ? 192 : 128;
        const uint32_t idesc = umma_idesc_bf16(256, n, 0, 1);
        for (int s = 0; s < 4; ++s)
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_2cta(tbase + (l & 1) * 256, desc(smem_u32(sA) + s * 16384 + kk * 32, 16, 1024, 2),
                           desc(smem_u32(sB) + s * 12288 + kk * 512, 2048, 256, 6), idesc, (s | kk) != 0);
      } else {
        const uint32_t idesc = umma_idesc_bf16(256, 96, 0, 1);
        for (int h = 0; h < 2; ++h)
          for (int s = 0; s < 4; ++s) {
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t bd = desc(smem_u32(sB) + s * 12288 + h * 6144 + kk * 512, 2048, 256, 6);
              if (mode == 1)
                umma_ts_2cta(tbase + 128 + h * 96, tbase + s * 32 + kk * 8, bd, idesc, (s | kk) != 0);
              else
                umma_bf16_2cta(tbase + 128 + h * 96, desc(smem_u32(sA) + s * 16384 + kk * 32, 16, 1024, 2), bd,
                               idesc, (s | kk) != 0);
            }
            if (mode == 1 && h == 1)
              for (int kk = 0; kk < 4; ++kk)
                utccp_2cta(tbase + s * 32 + kk * 8, desc(smem_u32(sA) + s * 16384 + kk * 32, 16, 1024, 2));
          }
      }
    }
    umma_commit_2cta(done, 0x3);
    mbar_wait(done, 0);
    cyc[blockIdx.x / 2] = clock64() - t0;
  } else {
    mbar_wait(done, 0);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc_2cta(tbase, 512);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap map2d(void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo, CUtensorMapSwizzle sw) {
  static EncodeFn enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    enc = reinterpret_cast<EncodeFn>(p);
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer}, str[1] = {inner * 2};
  cuuint32_t box[2] = {bi, bo}, es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}

static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return static_cast<uint16_t>((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}
static float bf2f(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

template <int N>
static int run() {
  const int M = 256;
  std::vector<uint16_t> a(M * K), b(K * N);
  srand(1);
  for (auto& x : a) x = f2bf((rand() / (float)RAND_MAX - 0.5f) * 4);
  for (auto& x : b) x = f2bf((rand() / (float)RAND_MAX - 0.5f) * 4);
  void *da, *db;
  float* dout;
  cudaMalloc(&da, a.size() * 2);
  cudaMalloc(&db, b.size() * 2);
  cudaMalloc(&dout, M * N * 4 * 2);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap tA = map2d(da, K, M, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tB = N == 128 ? map2d(db, N, K, 64, K, CU_TENSOR_MAP_SWIZZLE_128B)
                            : map2d(db, N, K, 16, K, CU_TENSOR_MAP_SWIZZLE_32B);
  auto kern = k_pair<N>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  std::vector<float> o[2];
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dout, 0, M * N * 4);
    kern<<<2, 128, 40000>>>(tA, tB, dout, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("N=%d mode %d: %s\n", N, mode, cudaGetErrorString(e));
      return 1;
    }
    o[mode].resize(M * N);
    cudaMemcpy(o[mode].data(), dout, M * N * 4, cudaMemcpyDeviceToHost);
  }
  double maxerr[2] = {0, 0};
  int same = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += (double)bf2f(a[i * K + k]) * bf2f(b[k * N + j]);
      for (int m = 0; m < 2; ++m) maxerr[m] = fmax(maxerr[m], fabs(o[m][i * N + j] - r));
      same += memcmp(&o[0][i * N + j], &o[1][i * N + j], 4) == 0;
    }
  printf("N=%d: SS max err %.3g, TS max err %.3g, TS == SS bitwise on %d / %d elements\n", N, maxerr[0], maxerr[1], same,
         M * N);
  return 0;
}

int main() {
  run<128>();
  run<96>();
  unsigned long long* dc;
  cudaMalloc(&dc, 8 * 74);
  cudaFuncSetAttribute(k_tput, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
  const int leaves = 2000;
  const char* names[4] = {"SS N=192 (16 MMAs/leaf)", "TS 2 x N=96 + 16 cp", "SS 2 x N=96 (A twice)", "SS N=128 (256x128 leaf)"};
  const double macs[4] = {256.0 * 192 * 256, 256.0 * 192 * 256, 256.0 * 192 * 256, 256.0 * 128 * 256};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) k_tput<<<148, 128, 120000>>>(leaves, mode, dc);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[74];
    cudaMemcpy(h, dc, 8 * 74, cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < 74; ++i) c += h[i];
    c /= 74;
    // pair peak: 8192 MAC/clk
    printf("%-28s %8.1f clk/leaf  %.3f of the pair MMA peak  (%s)\n", names[mode], c / leaves,
           macs[mode] / 8192.0 / (c / leaves), cudaGetErrorString(e));
  }
  return 0;
}
