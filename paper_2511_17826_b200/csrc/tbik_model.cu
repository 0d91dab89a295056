// tbik_model.cu -- the per-token kernels of a TBIK decoder forward:
// embedding gather, RoPE, causal GQA prefill attention, SiLU(gate) * up, and the
// residual add with the bf16 storage rounding of the reference demo
// (demo.cpp:36-81, 212-216).  Everything the tree GEMMs do not cover.
//
// Invariance: every output element is a fixed sequence of explicitly-rounded f32
// operations on inputs of its own token (and, for attention, its own sequence and
// head).  Nothing depends on the batch composition, on the TP sharding of heads /
// columns, or on the launch geometry -- so a forward built from these kernels,
// the TBIK GEMMs and the tree reductions is batch- and TP-invariant end to end.
// exp uses the shared polynomial of tbik_rowops.cu / oracle tbo_exp.
#include <string>

#include "tbik_common.cuh"
#include "tbik_internal.h"
#include "tbik_mathfn.cuh"

namespace tbik_b200 {

namespace {

__device__ __forceinline__ float bf(uint16_t b) { return bf16_bits_to_f32(b); }

// ---- embedding gather -------------------------------------------------------------
__global__ void embed_kernel(const uint16_t* __restrict__ table, int64_t H, const int64_t* __restrict__ ids,
                             int64_t V, uint16_t* __restrict__ out, int* __restrict__ bad) {
  const int64_t row = blockIdx.x;
  const int64_t id = ids[row];
  if (id < 0 || id >= V) {  // flagged; the row is zeroed so the output stays defined
    if (threadIdx.x == 0) *bad = 1;
    for (int64_t j = threadIdx.x; j < H; j += blockDim.x) out[row * H + j] = 0;
    return;
  }
  const uint16_t* src = table + id * H;
  uint16_t* dst = out + row * H;
  for (int64_t j = threadIdx.x; j < H; j += blockDim.x) dst[j] = src[j];
}

// ---- RoPE (rotate-half form) ----------------------------------------------------------
// x: f32 [M, ldx] columns [col0, col0 + heads*D); out bf16 [M, heads*D].
// out[d] = x[d]*cos - x[d+D/2]*sin (d < D/2), x[d]*cos + x[d-D/2]*sin (d >= D/2);
// optional per-head RMSNorm weight applied before (Qwen3 q/k norm) is done by the
// caller with tbik_tree_rmsnorm.
__global__ void rope_kernel(const float* __restrict__ x, int64_t ldx, int64_t col0, int heads, int D,
                            const int* __restrict__ pos, const float* __restrict__ cos_t,
                            const float* __restrict__ sin_t, uint16_t* __restrict__ out, int64_t ldo) {
  const int64_t row = blockIdx.x;
  const int p = pos[row];
  const int half = D / 2;
  const float* xr = x + row * ldx + col0;
  for (int e = threadIdx.x; e < heads * D; e += blockDim.x) {
    const int h = e / D, d = e - h * D;
    const float* xh = xr + h * D;
    float r;
    if (d < half) {
      const float c = cos_t[p * half + d], s = sin_t[p * half + d];
      r = __fsub_rn(__fmul_rn(xh[d], c), __fmul_rn(xh[d + half], s));
    } else {
      const float c = cos_t[p * half + d - half], s = sin_t[p * half + d - half];
      r = __fadd_rn(__fmul_rn(xh[d], c), __fmul_rn(xh[d - half], s));
    }
    out[row * ldo + e] = f32_to_bf16_bits(r);
  }
}

// f32 -> bf16 copy of a column block (V of qkv, storage casts).
__global__ void cast_kernel(const float* __restrict__ x, int64_t ldx, int64_t cols, uint16_t* __restrict__ out,
                            int64_t ldo) {
  const int64_t row = blockIdx.y;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[row * ldo + j] = f32_to_bf16_bits(x[row * ldx + j]);
}

// ---- causal GQA prefill attention, tiled two-pass form -------------------------------------
// Canonical order (restated in oracle tbo_attention_prefill), per (sequence, q head,
// query i), keys j = 0..i:
//   s_j = (ascending-d fma chain of q[d] k_j[d] from +0) * scale
//   m   = max_j s_j                                  (exact, order-free)
//   p_j = exp(s_j - m)                               (shared exp)
//   l   = ((p_0 + p_1) + p_2) + ...                  (ascending j)
//   o[d]= fma chain over ascending j of p_j v_j[d]   (from +0)
//   out = bf16(o[d] / l)
// One CTA = (32-query block, q head, sequence), 128 threads; K / V key blocks of
// 64 staged through shared memory as f32; scores for the whole causal prefix kept
// in shared memory (S <= 512).  Thread (i = t % 64, part = t / 64): 4 key phases in
// the score pass, 4 x 32-dim slices in the P.V pass; 4 independent fma chains each
// for ILP.  Per-query arithmetic never depends on the batch or the head sharding.
constexpr int AQ = 32;       // queries per CTA
constexpr int AK = 64;       // keys per staged block
constexpr int AD = 128;      // head dim
constexpr int AKP = AD + 4;  // padded f32 row of a staged K/V block

__global__ void __launch_bounds__(4 * AQ, 3) attn2_kernel(const uint16_t* __restrict__ q, int64_t ldq,
                                                    const uint16_t* __restrict__ k, int64_t ldk,
                                                    const uint16_t* __restrict__ v, int64_t ldv, int S, int nq,
                                                    int nkv, float scale, uint16_t* __restrict__ out, int64_t ldo) {
  extern __shared__ float sm[];
  float* kv = sm;                // [AK][AKP]
  float* P = sm + AK * AKP;      // [AQ][S + 1]
  float* red = P + AQ * (S + 1);  // [4][AQ] partial maxima, then l
  const int pst = S + 1;
  const int tid = threadIdx.x;
  const int qi = tid & (AQ - 1);
  const int part = tid / AQ;  // 0..3
  // grid (head, sequence, query block) with the query block slowest and reversed:
  // the heaviest (longest causal prefix) blocks are scheduled first and the light
  // ones fill the tail of the last wave.
  const int qb = static_cast<int>(gridDim.z) - 1 - static_cast<int>(blockIdx.z), h = blockIdx.x;
  const int64_t seq0 = static_cast<int64_t>(blockIdx.y) * S;
  const int kh = h / (nq / nkv);
  const int i = qb * AQ + qi;  // query position in the sequence
  const bool valid = i < S;
  const int last_key = min(S, (qb + 1) * AQ) - 1;  // keys needed by this block

  // q row in registers (f32).
  float qr[AD];
  {
    const uint16_t* qp = q + (seq0 + (valid ? i : 0)) * ldq + h * AD;
#pragma unroll
    for (int d = 0; d < AD; d += 8) {
      const uint4 raw = *reinterpret_cast<const uint4*>(qp + d);
      const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        qr[d + 2 * e] = __uint_as_float(w[e] << 16);
        qr[d + 2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
      }
    }
  }

  // ---- pass 1: scores ----
  for (int kb = 0; kb * AK <= last_key; ++kb) {
    __syncthreads();
    for (int e = tid; e < AK * AD / 8; e += blockDim.x) {  // stage K block as f32
      const int r = e / (AD / 8), c = (e % (AD / 8)) * 8;
      const int key = kb * AK + r;
      float* dst = kv + r * AKP + c;
      if (key <= last_key) {
        const uint4 raw = *reinterpret_cast<const uint4*>(k + (seq0 + key) * ldk + kh * AD + c);
        // two 16-byte stores (scalar stores at a 32-byte lane stride were 8-way bank conflicts)
        reinterpret_cast<float4*>(dst)[0] =
            make_float4(__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xFFFF0000u),
                        __uint_as_float(raw.y << 16), __uint_as_float(raw.y & 0xFFFF0000u));
        reinterpret_cast<float4*>(dst)[1] =
            make_float4(__uint_as_float(raw.z << 16), __uint_as_float(raw.z & 0xFFFF0000u),
                        __uint_as_float(raw.w << 16), __uint_as_float(raw.w & 0xFFFF0000u));
      }
    }
    __syncthreads();
    // keys jj = part + 4 * (4 r + u), u = 0..3 in flight together
#pragma unroll 1
    for (int r = 0; r < AK / 16; ++r) {
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      const float* kr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) kr[u] = kv + (part + 4 * (4 * r + u)) * AKP;
#pragma unroll
      for (int d = 0; d < AD; d += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 kk = *reinterpret_cast<const float4*>(kr[u] + d);
          acc[u] = __fmaf_rn(qr[d], kk.x, acc[u]);
          acc[u] = __fmaf_rn(qr[d + 1], kk.y, acc[u]);
          acc[u] = __fmaf_rn(qr[d + 2], kk.z, acc[u]);
          acc[u] = __fmaf_rn(qr[d + 3], kk.w, acc[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int key = kb * AK + part + 4 * (4 * r + u);
        if (key <= i && valid) P[qi * pst + key] = __fmul_rn(acc[u], scale);
      }
    }
  }
  __syncthreads();

  // ---- softmax: exact max, shared exp, ascending sum ----
  float mx = __int_as_float(0xFF800000);
  if (valid)
    for (int j = part; j <= i; j += 4) mx = fmaxf(mx, P[qi * pst + j]);
  red[part * AQ + qi] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(red[qi], red[AQ + qi]), fmaxf(red[2 * AQ + qi], red[3 * AQ + qi]));
  if (valid)
    for (int j = part; j <= i; j += 4) P[qi * pst + j] = tb_exp(__fsub_rn(P[qi * pst + j], mx));
  __syncthreads();
  if (part == 0) {
    float l = 0.0f;
    if (valid)
      for (int j = 0; j <= i; ++j) l = __fadd_rn(l, P[qi * pst + j]);
    red[qi] = l;
  }

  // ---- pass 2: o[d] = sum_j p_j v_j[d], dims [32 part, 32 part + 32) ----
  float o[32];
#pragma unroll
  for (int d = 0; d < 32; ++d) o[d] = 0.0f;
  const int d0 = part * 32;
  for (int kb = 0; kb * AK <= last_key; ++kb) {
    __syncthreads();
    for (int e = tid; e < AK * AD / 8; e += blockDim.x) {  // stage V block as f32
      const int r = e / (AD / 8), c = (e % (AD / 8)) * 8;
      const int key = kb * AK + r;
      float* dst = kv + r * AKP + c;
      if (key <= last_key) {
        const uint4 raw = *reinterpret_cast<const uint4*>(v + (seq0 + key) * ldv + kh * AD + c);
        // two 16-byte stores (scalar stores at a 32-byte lane stride were 8-way bank conflicts)
        reinterpret_cast<float4*>(dst)[0] =
            make_float4(__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xFFFF0000u),
                        __uint_as_float(raw.y << 16), __uint_as_float(raw.y & 0xFFFF0000u));
        reinterpret_cast<float4*>(dst)[1] =
            make_float4(__uint_as_float(raw.z << 16), __uint_as_float(raw.z & 0xFFFF0000u),
                        __uint_as_float(raw.w << 16), __uint_as_float(raw.w & 0xFFFF0000u));
      }
    }
    __syncthreads();
    const int jend = valid ? min(i, kb * AK + AK - 1) : -1;
    for (int j = kb * AK; j <= jend; ++j) {
      const float pj = P[qi * pst + j];
      const float* vr = kv + (j - kb * AK) * AKP + d0;
#pragma unroll
      for (int d = 0; d < 32; d += 4) {
        const float4 vv = *reinterpret_cast<const float4*>(vr + d);
        o[d] = __fmaf_rn(pj, vv.x, o[d]);
        o[d + 1] = __fmaf_rn(pj, vv.y, o[d + 1]);
        o[d + 2] = __fmaf_rn(pj, vv.z, o[d + 2]);
        o[d + 3] = __fmaf_rn(pj, vv.w, o[d + 3]);
      }
    }
  }
  __syncthreads();
  if (valid) {
    const float l = red[qi];
    uint16_t* op = out + (seq0 + i) * ldo + h * AD + d0;
#pragma unroll
    for (int d = 0; d < 32; d += 8) {
      uint32_t w[4];
#pragma unroll
      for (int x = 0; x < 4; ++x)
        w[x] = static_cast<uint32_t>(f32_to_bf16_bits(__fdiv_rn(o[d + 2 * x], l))) |
               (static_cast<uint32_t>(f32_to_bf16_bits(__fdiv_rn(o[d + 2 * x + 1], l))) << 16);
      *reinterpret_cast<uint4*>(op + d) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// ---- SiLU(gate) * up  (demo.cpp:36-45, :171-174) ---------------------------------------
// gu: f32 [M, ld] with gate in columns [0, I) and up in [I, 2I).  silu(z) = z / (1 + exp(-z)).
__device__ __forceinline__ uint16_t silu_mul1(float z, float up) { return tb_silu_mul_bf16(z, up); }

// Interleaved layout (gate_j at column 2j, up_j at 2j+1), the fallback of the
// fused gate_up GEMM (tbik_tree_matmul_silu_mul) when its epilogue cannot run.
__global__ void silu_mul_il_kernel(const float* __restrict__ gu, int64_t ld, int64_t I, uint16_t* __restrict__ out,
                                   int64_t ldo) {
  const int64_t row = blockIdx.y;
  const float* g = gu + row * ld;
  uint16_t* o = out + row * ldo;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < I;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    o[j] = silu_mul1(g[2 * j], g[2 * j + 1]);
}

// VEC: 4 consecutive columns per thread (16-byte loads, 8-byte stores).
template <bool VEC>
__global__ void silu_mul_kernel(const float* __restrict__ gu, int64_t ld, int64_t I, uint16_t* __restrict__ out,
                                int64_t ldo) {
  const int64_t row = blockIdx.y;
  const float* g = gu + row * ld;
  uint16_t* o = out + row * ldo;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (VEC) {
    for (int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; j < I; j += step * 4) {
      const float4 z = *reinterpret_cast<const float4*>(g + j);
      const float4 u = *reinterpret_cast<const float4*>(g + I + j);
      const uint32_t lo = silu_mul1(z.x, u.x) | (static_cast<uint32_t>(silu_mul1(z.y, u.y)) << 16);
      const uint32_t hi = silu_mul1(z.z, u.z) | (static_cast<uint32_t>(silu_mul1(z.w, u.w)) << 16);
      *reinterpret_cast<uint2*>(o + j) = make_uint2(lo, hi);
    }
  } else {
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < I; j += step)
      o[j] = silu_mul1(g[j], g[I + j]);
  }
}

// ---- residual: h = bf16(h + f)  (demo.cpp:216) -------------------------------------------------
template <bool VEC>
__global__ void residual_kernel(uint16_t* __restrict__ h, int64_t ldh, const float* __restrict__ f, int64_t ldf,
                                int64_t cols) {
  const int64_t row = blockIdx.y;
  uint16_t* hr = h + row * ldh;
  const float* fr = f + row * ldf;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (VEC) {
    for (int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; j < cols; j += step * 4) {
      const uint2 hv = *reinterpret_cast<const uint2*>(hr + j);
      const float4 fv = *reinterpret_cast<const float4*>(fr + j);
      const uint32_t lo = f32_to_bf16_bits(__fadd_rn(bf(hv.x & 0xFFFF), fv.x)) |
                          (static_cast<uint32_t>(f32_to_bf16_bits(__fadd_rn(bf(hv.x >> 16), fv.y))) << 16);
      const uint32_t hi = f32_to_bf16_bits(__fadd_rn(bf(hv.y & 0xFFFF), fv.z)) |
                          (static_cast<uint32_t>(f32_to_bf16_bits(__fadd_rn(bf(hv.y >> 16), fv.w))) << 16);
      *reinterpret_cast<uint2*>(hr + j) = make_uint2(lo, hi);
    }
  } else {
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols; j += step)
      hr[j] = f32_to_bf16_bits(__fadd_rn(bf(hr[j]), fr[j]));
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

tbik_status need_device() {
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  return TBIK_OK;
}

dim3 row_grid(int64_t rows, int64_t cols, int threads) {
  int64_t bx = (cols + threads - 1) / threads;
  if (bx > 64) bx = 64;
  return dim3(static_cast<unsigned>(bx), static_cast<unsigned>(rows));
}

}  // namespace

tbik_status launch_silu_mul_il(const float* gu, int64_t ld, int64_t rows, int64_t inter, uint16_t* out, int64_t ldo,
                               cudaStream_t s) {
  if (rows > 65535) return set_error(TBIK_BAD_DIMENSION, "silu_mul: bad dimensions");
  silu_mul_il_kernel<<<row_grid(rows, inter, 256), 256, 0, s>>>(gu, ld, inter, out, ldo);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

}  // namespace tbik_b200

using namespace tbik_b200;

extern "C" {

tbik_status tbik_embedding(const void* table, int64_t V, int64_t H, const int64_t* ids, int64_t rows, void* out,
                           void* stream) {
  if (!table || !ids || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || H < 1 || V < 1) return set_error(TBIK_BAD_DIMENSION, "embedding: dimensions must be >= 1");
  TBIK_TRY(need_device());
  int* bad = static_cast<int*>(workspace(16, 3));
  if (!bad) return set_error(TBIK_CUDA_ERROR, "workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TBIK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  embed_kernel<<<static_cast<unsigned>(rows), 256, 0, s>>>(static_cast<const uint16_t*>(table), H, ids, V,
                                                           static_cast<uint16_t*>(out), bad);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  // Out-of-range ids are reported synchronously (BadArgument) on an eager stream;
  // inside CUDA-graph capture no host sync is possible, so the check is skipped
  // (the kernel zeroes the row of such an id) -- callers validate ids before
  // capturing.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  TBIK_CUDA(cudaStreamIsCapturing(s, &cap));
  if (cap != cudaStreamCaptureStatusNone) return TBIK_OK;
  int hbad = 0;
  TBIK_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  TBIK_CUDA(cudaStreamSynchronize(s));
  if (hbad) return set_error(TBIK_BAD_ARGUMENT, "embedding: token id out of range");
  return TBIK_OK;
}

tbik_status tbik_rope(const float* x, int64_t ldx, int64_t col0, int heads, int head_dim, const int* positions,
                      const float* cos_table, const float* sin_table, void* out, int64_t ldo, int64_t rows,
                      void* stream) {
  if (!x || !positions || !cos_table || !sin_table || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (head_dim % 2 || heads < 1 || rows < 1) return set_error(TBIK_BAD_DIMENSION, "rope: bad dimensions");
  TBIK_TRY(need_device());
  rope_kernel<<<static_cast<unsigned>(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, ldx, col0, heads, head_dim, positions, cos_table, sin_table, static_cast<uint16_t*>(out), ldo);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_cast_bf16(const float* x, int64_t ldx, int64_t rows, int64_t cols, void* out, int64_t ldo,
                           void* stream) {
  if (!x || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || cols < 1 || rows > 65535) return set_error(TBIK_BAD_DIMENSION, "cast: bad dimensions");
  TBIK_TRY(need_device());
  cast_kernel<<<row_grid(rows, cols, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, ldx, cols, static_cast<uint16_t*>(out), ldo);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_attention_prefill(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                                   int64_t batch, int seq_len, int n_q_heads, int n_kv_heads, int head_dim,
                                   float scale, void* out, int64_t ldo, void* stream) {
  if (!q || !k || !v || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (head_dim != 128) return set_error(TBIK_UNSUPPORTED, "attention: head_dim must be 128");
  if (n_kv_heads < 1 || n_q_heads % n_kv_heads) return set_error(TBIK_BAD_DIMENSION, "attention: bad GQA heads");
  if (ldq % 4 || ldk % 4 || ldv % 4 || ldo % 4) return set_error(TBIK_BAD_ARGUMENT, "attention: strides % 4");
  if (seq_len < 1 || seq_len > 512) return set_error(TBIK_UNSUPPORTED, "attention: seq_len must be in [1, 512]");
  if (batch < 1 || batch > 65535 || n_q_heads > 65535) return set_error(TBIK_BAD_DIMENSION, "attention: grid");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
       reinterpret_cast<uintptr_t>(out)) & 15 || ldq % 8 || ldk % 8 || ldv % 8 || ldo % 8)
    return set_error(TBIK_BAD_ARGUMENT, "attention: 16-byte aligned rows required");
  TBIK_TRY(need_device());
  const size_t smem = (static_cast<size_t>(AK) * AKP + static_cast<size_t>(AQ) * (seq_len + 1) + 4 * AQ) * 4;
  static size_t attr = 0;
  if (attr < smem) {
    TBIK_CUDA(cudaFuncSetAttribute(attn2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr = smem;
  }
  dim3 grid(static_cast<unsigned>(n_q_heads), static_cast<unsigned>(batch),
            static_cast<unsigned>((seq_len + AQ - 1) / AQ));
  attn2_kernel<<<grid, 4 * AQ, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(q), ldq, static_cast<const uint16_t*>(k), ldk, static_cast<const uint16_t*>(v), ldv,
      seq_len, n_q_heads, n_kv_heads, scale, static_cast<uint16_t*>(out), ldo);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_silu_mul(const float* gate_up, int64_t ld, int64_t rows, int64_t inter, void* out, int64_t ldo,
                          void* stream) {
  if (!gate_up || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || inter < 1 || rows > 65535) return set_error(TBIK_BAD_DIMENSION, "silu_mul: bad dimensions");
  TBIK_TRY(need_device());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (inter % 4 == 0 && ld % 4 == 0 && ldo % 4 == 0 && aligned16(gate_up) && aligned16(out))
    silu_mul_kernel<true><<<row_grid(rows, inter / 4, 256), 256, 0, s>>>(gate_up, ld, inter,
                                                                        static_cast<uint16_t*>(out), ldo);
  else
    silu_mul_kernel<false><<<row_grid(rows, inter, 256), 256, 0, s>>>(gate_up, ld, inter,
                                                                     static_cast<uint16_t*>(out), ldo);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_residual_add(void* h, int64_t ldh, const float* f, int64_t ldf, int64_t rows, int64_t cols,
                              void* stream) {
  if (!h || !f) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || cols < 1 || rows > 65535) return set_error(TBIK_BAD_DIMENSION, "residual: bad dimensions");
  TBIK_TRY(need_device());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cols % 4 == 0 && ldh % 4 == 0 && ldf % 4 == 0 && aligned16(h) && aligned16(f))
    residual_kernel<true><<<row_grid(rows, cols / 4, 256), 256, 0, s>>>(static_cast<uint16_t*>(h), ldh, f, ldf, cols);
  else
    residual_kernel<false><<<row_grid(rows, cols, 256), 256, 0, s>>>(static_cast<uint16_t*>(h), ldh, f, ldf, cols);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

}  // extern "C"
