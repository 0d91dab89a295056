// tbik_rowops.cu -- tree-ordered RMSNorm and vocab-sharded log-softmax /
// log-prob (NEW semantics; the reference has only the sequential rmsnorm,
// demo.cpp:11-34, and softmax_row, demo.cpp:84-97).  The canonical orders are
// defined, and restated on the CPU, in oracle/tbik_oracle.c
// (tbo_tree_rmsnorm, tbo_tree_logsoftmax); this file must match it bit for bit.
//
// Both are HBM-bound row reductions: one 256-thread CTA per (row, vocab group),
// 16-byte loads, lane l folding chunks l, l+256, ... in ascending order, then
// a contiguous-halves tree: warp butterfly (xor 1, 2, 4, 8, 16 -- each level
// pairs adjacent subtrees, so it IS the contiguous-halves tree) and a fixed
// 8-warp tree through shared memory.
#include <math.h>

#include <algorithm>
#include <string>

#include "tbik_common.cuh"
#include "tbik_internal.h"
#include "tbik_mathfn.cuh"

namespace tbik_b200 {
namespace {

constexpr int LANES = 256;

// ---- (m, s) operator ---------------------------------------------------------
struct MS {
  float m, s;
};

__device__ __forceinline__ MS ms_merge(MS lo, MS hi) {
  if (lo.m == __int_as_float(0xFF800000)) return hi;
  if (hi.m == __int_as_float(0xFF800000)) return lo;
  const float m = lo.m >= hi.m ? lo.m : hi.m;
  const float a = __fmul_rn(lo.s, tb_exp_nonpos(__fsub_rn(lo.m, m)));  // arguments <= 0
  const float b = __fmul_rn(hi.s, tb_exp_nonpos(__fsub_rn(hi.m, m)));
  return MS{m, __fadd_rn(a, b)};
}

// Contiguous-halves tree over the 256 lane values of a CTA.
__device__ __forceinline__ float block_tree_sum(float v, float* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, d));
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  float r = 0.0f;
  if (threadIdx.x == 0) {
    const float a = __fadd_rn(sh[0], sh[1]), b = __fadd_rn(sh[2], sh[3]);
    const float c = __fadd_rn(sh[4], sh[5]), d = __fadd_rn(sh[6], sh[7]);
    r = __fadd_rn(__fadd_rn(a, b), __fadd_rn(c, d));
    sh[8] = r;
  }
  __syncthreads();
  return sh[8];
}

// ---- RMSNorm ------------------------------------------------------------------
// Pass 1 folds lane l's 16-byte chunks (l, l+256, ...) with an fma chain and
// keeps the first CACHE of them in registers; pass 2 revisits the same chunks
// with 16-byte loads of gamma and 16-byte stores (no second trip to memory for
// rows up to CACHE*256 chunks: 8192 bf16 / 4096 f32 columns).
template <typename TY>
__device__ __forceinline__ void store_chunk(TY* y, const float* r, int n);
template <>
__device__ __forceinline__ void store_chunk<float>(float* y, const float* r, int n) {
  if (n == 4) {
    *reinterpret_cast<float4*>(y) = make_float4(r[0], r[1], r[2], r[3]);
  } else if (n == 8) {
    *reinterpret_cast<float4*>(y) = make_float4(r[0], r[1], r[2], r[3]);
    *reinterpret_cast<float4*>(y + 4) = make_float4(r[4], r[5], r[6], r[7]);
  }
}
template <>
__device__ __forceinline__ void store_chunk<uint16_t>(uint16_t* y, const float* r, int n) {
  if (n == 8) {
    *reinterpret_cast<uint4*>(y) =
        make_uint4(bf16x2_bits(r[0], r[1]), bf16x2_bits(r[2], r[3]), bf16x2_bits(r[4], r[5]), bf16x2_bits(r[6], r[7]));
  } else if (n == 4) {
    *reinterpret_cast<uint2*>(y) = make_uint2(bf16x2_bits(r[0], r[1]), bf16x2_bits(r[2], r[3]));
  }
}

// (x * gamma) / denom, correctly rounded, with one reciprocal per row: q0 =
// RN(n * RN(1/d)), e = n - q0 * d (exact by fma), q = RN(q0 + e * RN(1/d)) is
// RN(n / d) (Markstein's theorem; no under/overflow in range, guarded).
__device__ __forceinline__ float div_rn_rcp(float n, float d, float rcp) {
  const float q0 = __fmul_rn(n, rcp);
  const float e = __fmaf_rn(-q0, d, n);
  const float q = __fmaf_rn(e, rcp, q0);
  const float aq = fabsf(q0);
  return (aq < 0x1p-100f || aq > 0x1p100f) ? __fdiv_rn(n, d) : q;
}

template <typename TX>
__device__ __forceinline__ float sumsq_chunk(const uint4& raw, float acc) {
  constexpr int CH = 16 / sizeof(TX);
  const TX* v = reinterpret_cast<const TX*>(&raw);
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const float f = load_as_f32(v + i);
    acc = __fmaf_rn(f, f, acc);
  }
  return acc;
}

template <typename TX, typename TY>
__device__ __forceinline__ void norm_chunk(const uint4& raw, const float* __restrict__ gamma, int64_t e0, float denom,
                                           float rcp, TY* y) {
  constexpr int CH = 16 / sizeof(TX);
  const TX* v = reinterpret_cast<const TX*>(&raw);
  float gm[CH], r[CH];
#pragma unroll
  for (int i = 0; i < CH; i += 4) *reinterpret_cast<float4*>(gm + i) = *reinterpret_cast<const float4*>(gamma + e0 + i);
  // div_rn_rcp with its range guard hoisted out of the element loop: the reciprocal
  // form for all CH elements, and -- rarely -- the whole chunk again by division
  // (in range both give RN(n / d), so the redo changes no in-range element)
  bool redo = false;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const float n = __fmul_rn(load_as_f32(v + i), gm[i]);
    const float q0 = __fmul_rn(n, rcp);
    const float e = __fmaf_rn(-q0, denom, n);
    r[i] = __fmaf_rn(e, rcp, q0);
    const float aq = fabsf(q0);
    redo |= aq < 0x1p-100f || aq > 0x1p100f;
  }
  if (redo) {
#pragma unroll
    for (int i = 0; i < CH; ++i) r[i] = __fdiv_rn(__fmul_rn(load_as_f32(v + i), gm[i]), denom);
  }
  store_chunk<TY>(y + e0, r, CH);
}

template <typename TX, typename TY, bool VEC>
__global__ void __launch_bounds__(LANES) tree_rmsnorm_kernel(const TX* __restrict__ X, int64_t ldx,
                                                             const float* __restrict__ gamma, float eps,
                                                             TY* __restrict__ Y, int64_t ldy, int64_t cols) {
  pdl_trigger();
  __shared__ float sh[9];
  constexpr int CH = 16 / sizeof(TX);  // 8 bf16 or 4 f32 per chunk
  constexpr int CACHE = 4;
  const TX* x = X + static_cast<int64_t>(blockIdx.x) * ldx;
  TY* y = Y + static_cast<int64_t>(blockIdx.x) * ldy;
  const int64_t nch = (cols + CH - 1) / CH;
  const int64_t nfull = cols / CH;  // chunks with CH valid elements
  float acc = 0.0f;
  if constexpr (VEC) {
    uint4 cache[CACHE];
#pragma unroll
    for (int k = 0; k < CACHE; ++k) {
      const int64_t c = threadIdx.x + static_cast<int64_t>(k) * LANES;
      if (c < nfull) cache[k] = *reinterpret_cast<const uint4*>(x + c * CH);
    }
    // pass 1: lane fold over chunks l, l+256, ... (cached ones first, same order)
#pragma unroll
    for (int k = 0; k < CACHE; ++k) {
      const int64_t c = threadIdx.x + static_cast<int64_t>(k) * LANES;
      if (c < nfull) acc = sumsq_chunk<TX>(cache[k], acc);
    }
    for (int64_t c = threadIdx.x + static_cast<int64_t>(CACHE) * LANES; c < nfull; c += LANES)
      acc = sumsq_chunk<TX>(*reinterpret_cast<const uint4*>(x + c * CH), acc);
    if (nfull < nch && threadIdx.x == nfull % LANES)  // ragged last chunk, in its lane's order
      for (int64_t e = nfull * CH; e < cols; ++e) {
        const float f = load_as_f32(x + e);
        acc = __fmaf_rn(f, f, acc);
      }
    const float ss = block_tree_sum(acc, sh);
    const float ms = __fdiv_rn(ss, static_cast<float>(cols));
    const float denom = __fsqrt_rn(__fadd_rn(ms, eps));
    const float rcp = __frcp_rn(denom);
    const bool yvec = (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (reinterpret_cast<uintptr_t>(gamma) & 15) == 0;
    if (yvec) {
#pragma unroll
      for (int k = 0; k < CACHE; ++k) {
        const int64_t c = threadIdx.x + static_cast<int64_t>(k) * LANES;
        if (c < nfull) norm_chunk<TX, TY>(cache[k], gamma, c * CH, denom, rcp, y);
      }
      for (int64_t c = threadIdx.x + static_cast<int64_t>(CACHE) * LANES; c < nfull; c += LANES)
        norm_chunk<TX, TY>(*reinterpret_cast<const uint4*>(x + c * CH), gamma, c * CH, denom, rcp, y);
    } else {
      for (int64_t e = threadIdx.x; e < nfull * CH; e += LANES) {
        const float r = div_rn_rcp(__fmul_rn(load_as_f32(x + e), gamma[e]), denom, rcp);
        if constexpr (sizeof(TY) == 4)
          y[e] = r;
        else
          y[e] = f32_to_bf16_bits(r);
      }
    }
    for (int64_t e = nfull * CH + threadIdx.x; e < cols; e += LANES) {
      const float r = div_rn_rcp(__fmul_rn(load_as_f32(x + e), gamma[e]), denom, rcp);
      if constexpr (sizeof(TY) == 4)
        y[e] = r;
      else
        y[e] = f32_to_bf16_bits(r);
    }
  } else {
    for (int64_t c = threadIdx.x; c < nch; c += LANES)
      for (int64_t e = c * CH; e < c * CH + CH && e < cols; ++e) {
        const float f = load_as_f32(x + e);
        acc = __fmaf_rn(f, f, acc);
      }
    const float ss = block_tree_sum(acc, sh);
    const float ms = __fdiv_rn(ss, static_cast<float>(cols));
    const float denom = __fsqrt_rn(__fadd_rn(ms, eps));
    const float rcp = __frcp_rn(denom);
    for (int64_t e = threadIdx.x; e < cols; e += LANES) {
      const float r = div_rn_rcp(__fmul_rn(load_as_f32(x + e), gamma[e]), denom, rcp);
      if constexpr (sizeof(TY) == 4)
        y[e] = r;
      else
        y[e] = f32_to_bf16_bits(r);
    }
  }
}

// h = bf16(h + f) (tbik_residual_add, demo.cpp:216) fused with the tree RMSNorm of
// the new h (bf16 -> bf16): the new row chunks are written back and kept in
// registers as the norm's cache, so the norm sees exactly the bits
// tree_rmsnorm_kernel would read.  cols % 8 == 0, cols <= CACHE * 256 * 8, 16-byte
// aligned rows (the launcher checks; otherwise it runs the two kernels).
__global__ void __launch_bounds__(LANES) residual_rmsnorm_kernel(uint16_t* __restrict__ Hm, int64_t ldh,
                                                                 const float* __restrict__ F, int64_t ldf,
                                                                 const float* __restrict__ gamma, float eps,
                                                                 uint16_t* __restrict__ Y, int64_t ldy, int64_t cols) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sh[9];
  constexpr int CH = 8;
  constexpr int CACHE = 4;
  uint16_t* h = Hm + static_cast<int64_t>(blockIdx.x) * ldh;
  const float* f = F + static_cast<int64_t>(blockIdx.x) * ldf;
  uint16_t* y = Y + static_cast<int64_t>(blockIdx.x) * ldy;
  const int64_t nfull = cols / CH;
  uint4 cache[CACHE];
#pragma unroll
  for (int k = 0; k < CACHE; ++k) {
    const int64_t c = threadIdx.x + static_cast<int64_t>(k) * LANES;
    if (c < nfull) {
      const uint4 hv = *reinterpret_cast<const uint4*>(h + c * CH);
      const float4 f0 = *reinterpret_cast<const float4*>(f + c * CH);
      const float4 f1 = *reinterpret_cast<const float4*>(f + c * CH + 4);
      uint4 nv;
      nv.x = f32_to_bf16_bits(__fadd_rn(bf16_bits_to_f32(hv.x & 0xFFFF), f0.x)) |
             (static_cast<uint32_t>(f32_to_bf16_bits(__fadd_rn(bf16_bits_to_f32(hv.x >> 16), f0.y))) << 16);
      nv.y = f32_to_bf16_bits(__fadd_rn(bf16_bits_to_f32(hv.y & 0xFFFF), f0.z)) |
             (static_cast<uint32_t>(f32_to_bf16_bits(__fadd_rn(bf16_bits_to_f32(hv.y >> 16), f0.w))) << 16);
      nv.z = f32_to_bf16_bits(__fadd_rn(bf16_bits_to_f32(hv.z & 0xFFFF), f1.x)) |
             (static_cast<uint32_t>(f32_to_bf16_bits(__fadd_rn(bf16_bits_to_f32(hv.z >> 16), f1.y))) << 16);
      nv.w = f32_to_bf16_bits(__fadd_rn(bf16_bits_to_f32(hv.w & 0xFFFF), f1.z)) |
             (static_cast<uint32_t>(f32_to_bf16_bits(__fadd_rn(bf16_bits_to_f32(hv.w >> 16), f1.w))) << 16);
      *reinterpret_cast<uint4*>(h + c * CH) = nv;
      cache[k] = nv;
    }
  }
  float acc = 0.0f;
#pragma unroll
  for (int k = 0; k < CACHE; ++k) {
    const int64_t c = threadIdx.x + static_cast<int64_t>(k) * LANES;
    if (c < nfull) acc = sumsq_chunk<uint16_t>(cache[k], acc);
  }
  const float ss = block_tree_sum(acc, sh);
  const float ms = __fdiv_rn(ss, static_cast<float>(cols));
  const float denom = __fsqrt_rn(__fadd_rn(ms, eps));
  const float rcp = __frcp_rn(denom);
#pragma unroll
  for (int k = 0; k < CACHE; ++k) {
    const int64_t c = threadIdx.x + static_cast<int64_t>(k) * LANES;
    if (c < nfull) norm_chunk<uint16_t, uint16_t>(cache[k], gamma, c * CH, denom, rcp, y);
  }
}

// ---- log-softmax ----------------------------------------------------------------
// Group states (tbo_tree_logsoftmax): one CTA per (row, group) of n = v_local /
// groups logits.  The group is cut into chunks of 16 logits from its start (the
// last possibly shorter); chunk c's (m, s) state is computed by thread c % 256
// from the logits (tb_ms_chunk16 -- the function the lm_head GEMM epilogue uses)
// or, FROM_STATES, read from a chunk-state array that epilogue (or
// chunk_states_kernel) wrote; the chunk states then meet by pairwise levels in
// shared memory ((2i, 2i+1) -> i, an odd last state passes up).
__device__ __forceinline__ MS chunk_state_mem(const float* __restrict__ x, int cnt, bool vec) {
  float v[TB_MS_CHUNK];
  if (vec && cnt == TB_MS_CHUNK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 f = reinterpret_cast<const float4*>(x)[q];
      v[4 * q] = f.x;
      v[4 * q + 1] = f.y;
      v[4 * q + 2] = f.z;
      v[4 * q + 3] = f.w;
    }
  } else {
    // a ragged chunk: -inf padding adds exp(-inf) = +0 terms (the sum is never -0)
    // and never wins the max -- the bits of the cnt-element chunk
#pragma unroll
    for (int k = 0; k < TB_MS_CHUNK; ++k) v[k] = k < cnt ? x[k] : __int_as_float(0xFF800000);
  }
  MS r;
  tb_ms_chunk16(v, r.m, r.s);
  return r;
}

template <bool FROM_STATES, bool VEC>
__global__ void __launch_bounds__(LANES) ms_group_kernel(const float* __restrict__ logits, int64_t ld, int64_t n,
                                                         const float2* __restrict__ chunks, int64_t ld_chunks,
                                                         int64_t groups, MS* __restrict__ out) {
  pdl_trigger();
  extern __shared__ MS ms_buf[];  // 2 x nc states (ping-pong)
  const int64_t row = blockIdx.x, g = blockIdx.y;
  const int nc = static_cast<int>((n + TB_MS_CHUNK - 1) / TB_MS_CHUNK);
  MS* a = ms_buf;
  MS* b = ms_buf + nc;
  for (int c = threadIdx.x; c < nc; c += LANES) {
    if constexpr (FROM_STATES) {
      const float2 f = chunks[row * ld_chunks + g * nc + c];
      a[c] = MS{f.x, f.y};
    } else {
      const int64_t e0 = static_cast<int64_t>(c) * TB_MS_CHUNK;
      const int cnt = n - e0 < TB_MS_CHUNK ? static_cast<int>(n - e0) : TB_MS_CHUNK;
      a[c] = chunk_state_mem(logits + row * ld + g * n + e0, cnt, VEC);
    }
  }
  __syncthreads();
  int cnt = nc;
  while (cnt > 1) {
    const int h = cnt >> 1;
    for (int i = threadIdx.x; i < h; i += LANES) b[i] = ms_merge(a[2 * i], a[2 * i + 1]);
    if ((cnt & 1) && threadIdx.x == 0) b[h] = a[cnt - 1];
    __syncthreads();
    MS* t = a;
    a = b;
    b = t;
    cnt = h + (cnt & 1);
  }
  if (threadIdx.x == 0) out[row * groups + g] = a[0];
}

// Chunk states of a [rows x v_local] logit block, groups of n (chunks restart at
// every group): the non-fused producer of the FROM_STATES input.
template <bool VEC>
__global__ void chunk_states_kernel(const float* __restrict__ logits, int64_t ld, int64_t n, int64_t groups,
                                    float2* __restrict__ out, int64_t ld_out) {
  pdl_trigger();
  const int64_t row = blockIdx.y;
  const int64_t nc = (n + TB_MS_CHUNK - 1) / TB_MS_CHUNK;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < groups * nc;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = i / nc, c = i - g * nc;
    const int64_t e0 = c * TB_MS_CHUNK;
    const int cnt = n - e0 < TB_MS_CHUNK ? static_cast<int>(n - e0) : TB_MS_CHUNK;
    const MS r = chunk_state_mem(logits + row * ld + g * n + e0, cnt, VEC);
    out[row * ld_out + i] = make_float2(r.m, r.s);
  }
}

// Contiguous-halves tree over `count` (power of two) states per row.
__device__ MS ms_tree(const MS* v, int64_t count) {
  // iterative binary counter (merge order lower, upper)
  MS stack[32];
  for (int64_t i = 0; i < count; ++i) {
    MS cur = v[i];
    int l = 0;
    uint64_t c = static_cast<uint64_t>(i);
    while (c & 1u) {
      cur = ms_merge(stack[l], cur);
      c >>= 1;
      ++l;
    }
    stack[l] = cur;
  }
  int j = 0;
  while ((int64_t{1} << j) < count) ++j;
  return stack[j];
}

__global__ void ms_rows_kernel(const MS* __restrict__ group_states, int64_t rows, int64_t groups,
                               float* __restrict__ ms_out) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const MS r = ms_tree(group_states + row * groups, groups);
  ms_out[2 * row] = r.m;
  ms_out[2 * row + 1] = r.s;
}

__global__ void ms_merge_kernel(PartPtrs parts, int W, int64_t rows, float* __restrict__ lse) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  MS v[kMaxRanks];
  for (int r = 0; r < W; ++r) v[r] = MS{parts.p[r][2 * row], parts.p[r][2 * row + 1]};
  const MS t = ms_tree(v, W);
  lse[row] = __fadd_rn(t.m, tb_log(t.s));
}

__global__ void finish_kernel(const float* __restrict__ logits, int64_t ld, int64_t rows, int64_t v_local,
                              const float* __restrict__ lse, float* __restrict__ logprobs, int64_t ld_out,
                              const int64_t* __restrict__ targets, int64_t v_offset, float* __restrict__ tlp,
                              bool vec) {
  pdl_trigger();
  const int64_t row = blockIdx.y;
  const float l = lse[row];
  if (logprobs) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (vec) {
      const float4* src = reinterpret_cast<const float4*>(logits + row * ld);
      float4* dst = reinterpret_cast<float4*>(logprobs + row * ld_out);
      for (int64_t j = t0; j < v_local / 4; j += stride) {
        const float4 q = src[j];
        dst[j] = make_float4(__fsub_rn(q.x, l), __fsub_rn(q.y, l), __fsub_rn(q.z, l), __fsub_rn(q.w, l));
      }
    } else {
      for (int64_t j = t0; j < v_local; j += stride) logprobs[row * ld_out + j] = __fsub_rn(logits[row * ld + j], l);
    }
  }
  if (targets && tlp && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t t = targets[row] - v_offset;
    if (t >= 0 && t < v_local) tlp[row] = __fsub_rn(logits[row * ld + t], l);
  }
}

}  // namespace
}  // namespace tbik_b200

using namespace tbik_b200;

extern "C" {

tbik_status tbik_tree_rmsnorm(const void* X, int x_dtype, int64_t ldx, const float* gamma, float eps, void* Y,
                              int y_dtype, int64_t ldy, int64_t rows, int64_t cols, void* stream) {
  if (!X || !Y || !gamma) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || cols < 1) return set_error(TBIK_BAD_DIMENSION, "rmsnorm: dimensions must be >= 1");
  if (ldx < cols || ldy < cols) return set_error(TBIK_BAD_ARGUMENT, "rmsnorm: leading dimension < cols");
  if ((x_dtype != TBIK_F32 && x_dtype != TBIK_BF16) || (y_dtype != TBIK_F32 && y_dtype != TBIK_BF16))
    return set_error(TBIK_UNKNOWN_DTYPE, "rmsnorm: dtype");
  if (rows > 0x7FFFFFFF) return set_error(TBIK_UNSUPPORTED, "rmsnorm: too many rows");
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t esz = x_dtype == TBIK_BF16 ? 2 : 4;
  const bool vec = (reinterpret_cast<uintptr_t>(X) & 15) == 0 && (ldx * esz) % 16 == 0;
  const unsigned g = static_cast<unsigned>(rows);
#define TBIK_RMS(TX, TY)                                                                                   \
  (vec ? (tree_rmsnorm_kernel<TX, TY, true><<<g, LANES, 0, s>>>(static_cast<const TX*>(X), ldx, gamma, eps,  \
                                                                static_cast<TY*>(Y), ldy, cols),             \
          0)                                                                                                 \
       : (tree_rmsnorm_kernel<TX, TY, false><<<g, LANES, 0, s>>>(static_cast<const TX*>(X), ldx, gamma, eps, \
                                                                 static_cast<TY*>(Y), ldy, cols),            \
          0))
  if (x_dtype == TBIK_BF16 && y_dtype == TBIK_F32) TBIK_RMS(uint16_t, float);
  else if (x_dtype == TBIK_BF16) TBIK_RMS(uint16_t, uint16_t);
  else if (y_dtype == TBIK_F32) TBIK_RMS(float, float);
  else TBIK_RMS(float, uint16_t);
#undef TBIK_RMS
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_residual_rmsnorm(void* h, int64_t ldh, const float* f, int64_t ldf, const float* gamma, float eps,
                                  void* y, int64_t ldy, int64_t rows, int64_t cols, void* stream) {
  if (!h || !f || !gamma || !y) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || cols < 1) return set_error(TBIK_BAD_DIMENSION, "residual_rmsnorm: dimensions must be >= 1");
  if (ldh < cols || ldf < cols || ldy < cols) return set_error(TBIK_BAD_ARGUMENT, "residual_rmsnorm: leading dimension < cols");
  if (rows > 0x7FFFFFFF) return set_error(TBIK_UNSUPPORTED, "residual_rmsnorm: too many rows");
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (cols % 8 == 0 && cols <= 4 * LANES * 8 && ldh % 8 == 0 && ldf % 4 == 0 && ldy % 8 == 0 && a16(h) && a16(f) &&
      a16(y) && a16(gamma)) {
    if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
    TBIK_CUDA(launch_pdl(residual_rmsnorm_kernel, dim3(static_cast<unsigned>(rows)), dim3(LANES), 0,
                         static_cast<cudaStream_t>(stream), static_cast<uint16_t*>(h), ldh, f, ldf, gamma, eps,
                         static_cast<uint16_t*>(y), ldy, cols));
    TBIK_CUDA(cudaGetLastError());
    count_launch();
    return TBIK_OK;
  }
  // unfused: the same two kernels back to back (same bits)
  const tbik_status st = tbik_residual_add(h, ldh, f, ldf, rows, cols, stream);
  if (st != TBIK_OK) return st;
  return tbik_tree_rmsnorm(h, TBIK_BF16, ldh, gamma, eps, y, TBIK_BF16, ldy, rows, cols, stream);
}

namespace {
tbik_status shard_state_impl(const float* logits, int64_t ld, const float2* chunks, int64_t ld_chunks, int64_t rows,
                             int64_t v_local, int64_t groups, float* ms_out, cudaStream_t s) {
  if (!ms_out || (!logits && !chunks)) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || v_local < 1) return set_error(TBIK_BAD_DIMENSION, "logsoftmax: dimensions must be >= 1");
  if (groups < 1 || (groups & (groups - 1)) || v_local % groups)
    return set_error(TBIK_SHARD_ERROR, "logsoftmax: shard of " + std::to_string(v_local) +
                                           " logits is not a power-of-two number of equal groups (" +
                                           std::to_string(groups) + ")");
  if (logits && ld < v_local) return set_error(TBIK_BAD_ARGUMENT, "logsoftmax: ld < v_local");
  if (rows > 0x7FFFFFFF || groups > 65535) return set_error(TBIK_UNSUPPORTED, "logsoftmax: grid too large");
  const int64_t n = v_local / groups;
  const int64_t nc = (n + TB_MS_CHUNK - 1) / TB_MS_CHUNK;
  const size_t smem = static_cast<size_t>(2 * nc) * sizeof(MS);
  if (chunks && ld_chunks < groups * nc) return set_error(TBIK_BAD_ARGUMENT, "logsoftmax: ld_chunks too small");
  if (smem > 200 * 1024)
    return set_error(TBIK_UNSUPPORTED, "logsoftmax: vocab group of " + std::to_string(n) +
                                           " logits exceeds one CTA's chunk buffer; use more groups");
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  MS* gs = static_cast<MS*>(workspace(static_cast<size_t>(rows) * groups * sizeof(MS), 3, s));
  if (!gs) return set_error(TBIK_CUDA_ERROR, "workspace allocation failed");
  const bool vec = logits && (reinterpret_cast<uintptr_t>(logits) & 15) == 0 && ld % 4 == 0 && n % 4 == 0;
  dim3 grid(static_cast<unsigned>(rows), static_cast<unsigned>(groups));
  auto kern = chunks ? ms_group_kernel<true, false> : vec ? ms_group_kernel<false, true> : ms_group_kernel<false, false>;
  if (smem > 48 * 1024)
    TBIK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<grid, LANES, smem, s>>>(logits, ld, n, chunks, ld_chunks, groups, gs);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  ms_rows_kernel<<<static_cast<unsigned>((rows + 127) / 128), 128, 0, s>>>(gs, rows, groups, ms_out);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}
}  // namespace

tbik_status tbik_logsoftmax_shard_state(const float* logits, int64_t ld, int64_t rows, int64_t v_local, int64_t groups,
                                        float* ms_out, void* stream) {
  if (!logits) return set_error(TBIK_BAD_ARGUMENT, "null logits");
  return shard_state_impl(logits, ld, nullptr, 0, rows, v_local, groups, ms_out, static_cast<cudaStream_t>(stream));
}

tbik_status tbik_logsoftmax_shard_state_chunks(const float* chunk_ms, int64_t ld_chunks, int64_t rows, int64_t v_local,
                                               int64_t groups, float* ms_out, void* stream) {
  if (!chunk_ms) return set_error(TBIK_BAD_ARGUMENT, "null chunk states");
  if (reinterpret_cast<uintptr_t>(chunk_ms) & 7) return set_error(TBIK_BAD_ARGUMENT, "chunk states: 8-byte alignment");
  return shard_state_impl(nullptr, 0, reinterpret_cast<const float2*>(chunk_ms), ld_chunks, rows, v_local, groups,
                          ms_out, static_cast<cudaStream_t>(stream));
}

tbik_status tbik_logsoftmax_chunk_states(const float* logits, int64_t ld, int64_t rows, int64_t v_local,
                                         int64_t groups, float* chunk_ms, int64_t ld_chunks, void* stream) {
  if (!logits || !chunk_ms) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || v_local < 1) return set_error(TBIK_BAD_DIMENSION, "logsoftmax: dimensions must be >= 1");
  if (groups < 1 || (groups & (groups - 1)) || v_local % groups)
    return set_error(TBIK_SHARD_ERROR, "logsoftmax: groups must be a power of two dividing the shard");
  if (ld < v_local) return set_error(TBIK_BAD_ARGUMENT, "logsoftmax: ld < v_local");
  if (rows > 65535) return set_error(TBIK_UNSUPPORTED, "logsoftmax: > 65535 rows per call");
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  const int64_t n = v_local / groups, nc = (n + TB_MS_CHUNK - 1) / TB_MS_CHUNK;
  if (ld_chunks < groups * nc) return set_error(TBIK_BAD_ARGUMENT, "logsoftmax: ld_chunks too small");
  if (reinterpret_cast<uintptr_t>(chunk_ms) & 7) return set_error(TBIK_BAD_ARGUMENT, "chunk states: 8-byte alignment");
  const bool vec = (reinterpret_cast<uintptr_t>(logits) & 15) == 0 && ld % 4 == 0 && n % 4 == 0;
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((groups * nc + 255) / 256, 64)), static_cast<unsigned>(rows));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (vec)
    chunk_states_kernel<true><<<grid, 256, 0, s>>>(logits, ld, n, groups, reinterpret_cast<float2*>(chunk_ms),
                                                   ld_chunks);
  else
    chunk_states_kernel<false><<<grid, 256, 0, s>>>(logits, ld, n, groups, reinterpret_cast<float2*>(chunk_ms),
                                                    ld_chunks);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_logsoftmax_merge(const float* const* ms_parts, int W, int64_t rows, float* lse, void* stream) {
  if (!ms_parts || !lse) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (W < 1 || (W & (W - 1)) || W > kMaxRanks) return set_error(TBIK_BAD_WORLD_SIZE, "world size must be a power of two");
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  PartPtrs pp{};
  for (int r = 0; r < W; ++r) pp.p[r] = ms_parts[r];
  ms_merge_kernel<<<static_cast<unsigned>((rows + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(pp, W, rows,
                                                                                                        lse);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_logsoftmax_finish(const float* logits, int64_t ld, int64_t rows, int64_t v_local, const float* lse,
                                   float* logprobs, int64_t ld_out, const int64_t* targets, int64_t v_offset,
                                   float* target_logprobs, void* stream) {
  if (!logits || !lse) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows > 65535) return set_error(TBIK_UNSUPPORTED, "logsoftmax finish: > 65535 rows per call");
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  const bool vec = logprobs && (reinterpret_cast<uintptr_t>(logits) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(logprobs) & 15) == 0 && ld % 4 == 0 && ld_out % 4 == 0 &&
                   v_local % 4 == 0;
  const int64_t xblocks = logprobs ? std::min<int64_t>((v_local + 4095) / 4096, 16) : 1;
  dim3 grid(static_cast<unsigned>(xblocks), static_cast<unsigned>(rows));
  finish_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(logits, ld, rows, v_local, lse, logprobs, ld_out,
                                                                     targets, v_offset, target_logprobs, vec);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_tree_logsoftmax_local(const float* logits, int64_t ld, int64_t rows, int64_t V, int64_t groups, int tp,
                                       float* lse, float* logprobs, int64_t ld_out, const int64_t* targets,
                                       float* target_logprobs, void* stream) {
  if (tp < 1 || (tp & (tp - 1)) || tp > kMaxRanks) return set_error(TBIK_BAD_WORLD_SIZE, "tp must be a power of two");
  if (V % tp || groups % tp)
    return set_error(TBIK_SHARD_ERROR, "vocab / groups not divisible by tp=" + std::to_string(tp));
  const int64_t vl = V / tp;
  float* ms = static_cast<float*>(workspace(static_cast<size_t>(rows) * 2 * tp * sizeof(float), 2, static_cast<cudaStream_t>(stream)));
  if (!ms) return set_error(TBIK_CUDA_ERROR, "workspace allocation failed");
  PartPtrs pp{};
  for (int r = 0; r < tp; ++r) {
    TBIK_TRY(tbik_logsoftmax_shard_state(logits + r * vl, ld, rows, vl, groups / tp, ms + 2 * rows * r, stream));
    pp.p[r] = ms + 2 * rows * r;
  }
  TBIK_TRY(tbik_logsoftmax_merge(pp.p, tp, rows, lse, stream));
  for (int r = 0; r < tp; ++r)
    TBIK_TRY(tbik_logsoftmax_finish(logits + r * vl, ld, rows, vl, lse, logprobs ? logprobs + r * vl : nullptr,
                                    ld_out, targets, r * vl, target_logprobs, stream));
  return TBIK_OK;
}

}  // extern "C"
