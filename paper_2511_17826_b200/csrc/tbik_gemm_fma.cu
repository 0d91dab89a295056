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
  count_launch();
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
  if (v.adt == TBIK_BF16 && v.bdt == TBIK_BF16) return launch_typed<uint16_t, uint16_t>(v, o, s);
  if (v.adt == TBIK_BF16 && v.bdt == TBIK_F32) return launch_typed<uint16_t, float>(v, o, s);
  if (v.adt == TBIK_F32 && v.bdt == TBIK_BF16) return launch_typed<float, uint16_t>(v, o, s);
  return launch_typed<float, float>(v, o, s);
}

}  // namespace tbik_b200
