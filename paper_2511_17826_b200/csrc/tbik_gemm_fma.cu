// tbik_gemm_fma.cu -- the EXACT-LEAF TBIK GEMM on CUDA cores.
//
// Leaf semantics are the reference's leaf_dot (matmul.cpp:69-75) verbatim:
// for every output element, an ascending-k __fmaf_rn chain from +0 over the
// tile's K extent (ragged tail tiles simply do fewer fmas, matmul.cpp:177-178).
// Operands are widened bf16 -> f32 exactly (bits << 16, numerics.hpp:44-46).
// The launch produces either one f32 slice per leaf tile (OUT_LEAVES) or one
// per leaf group with the level-0 fold done in-register (OUT_GROUPS:
// g = ((0 + P_0) + P_1) + ..., TileReducer level 0, matmul.cpp:100-125); the
// tree above is tbik_tree.cu's combine.  Output tiling (BM x BN) never touches
// the per-element operation sequence, so any tiling gives identical bits --
// that is what lets the launcher choose tiles by M without breaking batch
// invariance.
#include <cstdlib>
#include <string>

#include "tbik_common.cuh"
#include "tbik_internal.h"

namespace tbik_b200 {

namespace {

constexpr int KC = 32;  // K chunk staged through shared memory

template <int BM, int BN, int TM, int TN, typename TA, typename TB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    fma_tree_gemm_kernel(const TA* __restrict__ A, int64_t lda, const TB* __restrict__ B, int64_t ldb,
                         int64_t M, int64_t N, int64_t K, int64_t bk, int64_t kf, int64_t T,
                         int mode, float* __restrict__ out, int64_t ldo, int64_t unit_stride) {
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int TX = BN / TN;
  __shared__ float As[KC][BM];
  __shared__ float Bs[KC][BN];

  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
  const int64_t unit = blockIdx.z;
  const int64_t tiles_per_unit = mode == OUT_LEAVES ? 1 : kf;
  const int64_t t_begin = unit * tiles_per_unit;
  const int64_t t_end = t_begin + tiles_per_unit < T ? t_begin + tiles_per_unit : T;

  float g[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) g[i][j] = 0.0f;

  for (int64_t t = t_begin; t < t_end; ++t) {
    const int64_t kt0 = t * bk;
    const int64_t kt1 = kt0 + bk < K ? kt0 + bk : K;
    float p[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) p[i][j] = 0.0f;

    for (int64_t kc0 = kt0; kc0 < kt1; kc0 += KC) {
      const int kcn = static_cast<int>(kt1 - kc0 < KC ? kt1 - kc0 : KC);
      // Stage A[m0:m0+BM, kc0:kc0+kcn] transposed and B[kc0:, n0:n0+BN].
      for (int idx = tid; idx < BM * KC; idx += NT) {
        const int mm = idx / KC, kk = idx % KC;
        const int64_t gm = m0 + mm;
        As[kk][mm] = (kk < kcn && gm < M) ? load_as_f32(A + gm * lda + kc0 + kk) : 0.0f;
      }
      for (int idx = tid; idx < BN * KC; idx += NT) {
        const int kk = idx / BN, nn = idx % BN;
        const int64_t gn = n0 + nn;
        Bs[kk][nn] = (kk < kcn && gn < N) ? load_as_f32(B + (kc0 + kk) * ldb + gn) : 0.0f;
      }
      __syncthreads();
      // Ascending k, one fma per element per k: exactly leaf_dot's chain.
      for (int kk = 0; kk < kcn; ++kk) {
        float a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx * TN + j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) p[i][j] = __fmaf_rn(a[i], b[j], p[i][j]);
      }
      __syncthreads();
    }

    if (mode == OUT_LEAVES) {
      float* dst = out + t * unit_stride;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int64_t gm = m0 + ty * TM + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const int64_t gn = n0 + tx * TN + j;
          if (gn < N) dst[gm * ldo + gn] = p[i][j];
        }
      }
    } else {
      // Level-0 fold: g = g + P (g starts at +0, so the first add canonicalises).
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) g[i][j] = __fadd_rn(g[i][j], p[i][j]);
    }
  }

  if (mode == OUT_GROUPS) {
    float* dst = out + unit * unit_stride;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t gm = m0 + ty * TM + i;
      if (gm >= M) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t gn = n0 + tx * TN + j;
        if (gn < N) dst[gm * ldo + gn] = g[i][j];
      }
    }
  }
}

// ---- v2: bf16 x bf16, 128 x 128 tiles, 16-byte loads, double-buffered K chunks ----
// Same per-element chain as fma_tree_gemm_kernel (ascending k, one __fmaf_rn per
// k, restart at each leaf tile; the ragged tail tile runs exactly kcn fmas).  A
// thread owns rows {4ty..4ty+3, 64+4ty..} x columns {4tx..4tx+3, 64+4tx..} so its
// shared-memory reads are conflict-free 16-byte vectors; the next K chunk is
// fetched into registers while the current one is consumed.
constexpr int V2_KC = 32;
constexpr int V2_SMEM = 2 * 2 * V2_KC * 128 * 4;  // two buffers of A^T and B chunks (64 KB)

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    f[2 * e] = __uint_as_float(w[e] << 16);
    f[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
  }
}

__global__ void __launch_bounds__(256, 1)
    fma_tree_gemm_v2(const uint16_t* __restrict__ A, int64_t lda, const uint16_t* __restrict__ B, int64_t ldb,
                     int64_t M, int64_t N, int64_t K, int64_t bk, int64_t kf, int64_t T, int mode,
                     float* __restrict__ out, int64_t ldo, int64_t unit_stride) {
  extern __shared__ float v2_sm[];
  float* As = v2_sm;                       // [2][KC][128]  (A transposed: k-major)
  float* Bs = v2_sm + 2 * V2_KC * 128;     // [2][KC][128]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * 128;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * 128;
  const int64_t unit = blockIdx.z;
  const int64_t tiles_per_unit = mode == OUT_LEAVES ? 1 : kf;
  const int64_t t_begin = unit * tiles_per_unit;
  const int64_t t_end = t_begin + tiles_per_unit < T ? t_begin + tiles_per_unit : T;
  // loader roles: threads 0-127 stage A (k-octet ko, rows 4rq..4rq+3),
  // threads 128-255 stage B (k rows kb + 8j, columns 8no..8no+7)
  const bool ldA = tid < 128;
  const int ko = (tid & 127) >> 5, rq = tid & 31;
  const int no = tid & 15, kb = (tid & 127) >> 4;
  uint4 reg[4];

  auto gload = [&](int64_t kc0, int64_t kt1) {
    if (ldA) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t gm = m0 + 4 * rq + j, gk = kc0 + 8 * ko;
        reg[j] = (gm < M && gk < kt1) ? *reinterpret_cast<const uint4*>(A + gm * lda + gk) : make_uint4(0, 0, 0, 0);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t gk = kc0 + kb + 8 * j, gn = n0 + 8 * no;
        reg[j] = (gk < kt1 && gn < N) ? *reinterpret_cast<const uint4*>(B + gk * ldb + gn) : make_uint4(0, 0, 0, 0);
      }
    }
  };
  auto sstore = [&](int buf) {
    if (ldA) {
      float f[4][8];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf16x8_to_f32(reg[j], f[j]);
      float* dst = As + (buf * V2_KC + 8 * ko) * 128 + 4 * rq;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        *reinterpret_cast<float4*>(dst + e * 128) = make_float4(f[0][e], f[1][e], f[2][e], f[3][e]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float f[8];
        bf16x8_to_f32(reg[j], f);
        float* dst = Bs + (buf * V2_KC + kb + 8 * j) * 128 + 8 * no;
        *reinterpret_cast<float4*>(dst) = make_float4(f[0], f[1], f[2], f[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(f[4], f[5], f[6], f[7]);
      }
    }
  };

  float g[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) g[i][j] = 0.0f;

  for (int64_t t = t_begin; t < t_end; ++t) {
    const int64_t kt0 = t * bk;
    const int64_t kt1 = kt0 + bk < K ? kt0 + bk : K;
    float p[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) p[i][j] = 0.0f;
    int buf = 0;
    gload(kt0, kt1);
    __syncthreads();  // the previous tile's last chunk is consumed
    sstore(0);
    __syncthreads();
    for (int64_t kc0 = kt0; kc0 < kt1; kc0 += V2_KC) {
      const int kcn = static_cast<int>(kt1 - kc0 < V2_KC ? kt1 - kc0 : V2_KC);
      const bool more = kc0 + V2_KC < kt1;
      if (more) gload(kc0 + V2_KC, kt1);
      const float* a_s = As + buf * V2_KC * 128;
      const float* b_s = Bs + buf * V2_KC * 128;
      for (int kk = 0; kk < kcn; ++kk) {  // ascending k: exactly leaf_dot's chain
        const float4 a0 = *reinterpret_cast<const float4*>(a_s + kk * 128 + 4 * ty);
        const float4 a1 = *reinterpret_cast<const float4*>(a_s + kk * 128 + 64 + 4 * ty);
        const float4 b0 = *reinterpret_cast<const float4*>(b_s + kk * 128 + 4 * tx);
        const float4 b1 = *reinterpret_cast<const float4*>(b_s + kk * 128 + 64 + 4 * tx);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) p[i][j] = __fmaf_rn(a[i], b[j], p[i][j]);
      }
      if (more) sstore(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
    if (mode == OUT_LEAVES) {
      float* dst = out + t * unit_stride;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t gm = m0 + (i < 4 ? 4 * ty + i : 64 + 4 * ty + i - 4);
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int64_t gn = n0 + (j < 4 ? 4 * tx + j : 64 + 4 * tx + j - 4);
          if (gn < N) dst[gm * ldo + gn] = p[i][j];
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) g[i][j] = __fadd_rn(g[i][j], p[i][j]);  // level-0 fold
    }
  }
  if (mode == OUT_GROUPS) {
    float* dst = out + unit * unit_stride;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t gm = m0 + (i < 4 ? 4 * ty + i : 64 + 4 * ty + i - 4);
      if (gm >= M) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t gn = n0 + (j < 4 ? 4 * tx + j : 64 + 4 * tx + j - 4);
        if (gn < N) dst[gm * ldo + gn] = g[i][j];
      }
    }
  }
}

tbik_status launch_v2(const GemmView& v, const GemmOut& o, cudaStream_t s) {
  const int64_t units = o.mode == OUT_LEAVES ? v.T : v.L;
  dim3 grid(static_cast<unsigned>((v.N + 127) / 128), static_cast<unsigned>((v.M + 127) / 128),
            static_cast<unsigned>(units));
  if (grid.y > 65535 || grid.z > 65535) return set_error(TBIK_UNSUPPORTED, "fma gemm: grid too large");
  // per launch: the attribute belongs to the current device's context (a host call
  // of ~1 us, next to a kernel of >= 10 us)
  TBIK_CUDA(cudaFuncSetAttribute(fma_tree_gemm_v2, cudaFuncAttributeMaxDynamicSharedMemorySize, V2_SMEM));
  fma_tree_gemm_v2<<<grid, 256, V2_SMEM, s>>>(static_cast<const uint16_t*>(v.A), v.lda,
                                              static_cast<const uint16_t*>(v.B), v.ldb, v.M, v.N, v.K, v.bk, v.kf,
                                              v.T, o.mode, o.out, o.ldo, o.unit_stride);
  TBIK_CUDA(cudaGetLastError());
  count_launch("fma_tree_gemm_v2");
  return TBIK_OK;
}

template <int BM, int BN, int TM, int TN, typename TA, typename TB>
tbik_status launch_cfg(const GemmView& v, const GemmOut& o, cudaStream_t s) {
  const int64_t units = o.mode == OUT_LEAVES ? v.T : v.L;
  dim3 grid(static_cast<unsigned>((v.N + BN - 1) / BN), static_cast<unsigned>((v.M + BM - 1) / BM),
            static_cast<unsigned>(units));
  if (grid.y > 65535 || grid.z > 65535)
    return set_error(TBIK_UNSUPPORTED, "fma gemm: grid too large");
  fma_tree_gemm_kernel<BM, BN, TM, TN, TA, TB><<<grid, (BM / TM) * (BN / TN), 0, s>>>(
      static_cast<const TA*>(v.A), v.lda, static_cast<const TB*>(v.B), v.ldb, v.M, v.N, v.K, v.bk,
      v.kf, v.T, o.mode, o.out, o.ldo, o.unit_stride);
  TBIK_CUDA(cudaGetLastError());
  count_launch("fma_tree_gemm_kernel");
  return TBIK_OK;
}

template <typename TA, typename TB>
tbik_status launch_typed(const GemmView& v, const GemmOut& o, cudaStream_t s) {
  // Tile choice by M is a pure scheduling decision (see file comment).
  if (v.M <= 8) return launch_cfg<8, 128, 1, 4, TA, TB>(v, o, s);
  if (v.M <= 32) return launch_cfg<32, 128, 4, 4, TA, TB>(v, o, s);
  return launch_cfg<128, 128, 8, 8, TA, TB>(v, o, s);
}

}  // namespace

tbik_status launch_fma_gemm(const GemmView& v, const GemmOut& o, cudaStream_t s) {
  if (o.mode != OUT_LEAVES && o.mode != OUT_GROUPS)
    return set_error(TBIK_BAD_ARGUMENT, "fma gemm: mode must be LEAVES or GROUPS");
  if (v.adt == TBIK_BF16 && v.bdt == TBIK_BF16) {
    // v2 needs 16-byte rows and chunks: K, N, lda, ldb multiples of 8, aligned bases,
    // block_k a multiple of its 32-wide K chunk (a pure scheduling choice: same bits).
    const bool v2 = v.M > 32 && v.K % 8 == 0 && v.N % 8 == 0 && v.lda % 8 == 0 && v.ldb % 8 == 0 &&
                    v.bk % V2_KC == 0 && (reinterpret_cast<uintptr_t>(v.A) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(v.B) & 15) == 0 && knob(KNOB_FMA_V1, 0) == 0;
    if (v2) return launch_v2(v, o, s);
    return launch_typed<uint16_t, uint16_t>(v, o, s);
  }
  if (v.adt == TBIK_BF16 && v.bdt == TBIK_F32) return launch_typed<uint16_t, float>(v, o, s);
  if (v.adt == TBIK_F32 && v.bdt == TBIK_BF16) return launch_typed<float, uint16_t>(v, o, s);
  return launch_typed<float, float>(v, o, s);
}

}  // namespace tbik_b200
