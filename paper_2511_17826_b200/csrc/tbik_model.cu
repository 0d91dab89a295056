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
  if (id < 0 || id >= V) {
    if (threadIdx.x == 0) *bad = 1;
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

// ---- causal GQA prefill attention ---------------------------------------------------------
// One warp per (sequence, q head, query).  Lane l owns head dims [4l, 4l+4) (D = 128).
// score_j = T(lane partial fma chains) * scale   (T = contiguous-halves butterfly)
// online softmax over keys j = 0..i ascending with the shared exp:
//   s > m: a = exp(m - s); l = l*a + 1; o = o*a + v_j; m = s
//   else : p = exp(s - m); l = l + p;   o = fma(p, v_j, o)
// out = o / l, rounded to bf16.  Fixed order per (seq, head, query): batch- and
// TP-(head-sharding-)invariant.
__global__ void __launch_bounds__(256) attn_kernel(const uint16_t* __restrict__ q, int64_t ldq,
                                                   const uint16_t* __restrict__ k, int64_t ldk,
                                                   const uint16_t* __restrict__ v, int64_t ldv, int S, int nq,
                                                   int nkv, float scale, uint16_t* __restrict__ out, int64_t ldo,
                                                   int64_t total_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  // gw enumerates (row = token, head)
  const int64_t row = gw / nq;
  const int h = static_cast<int>(gw - row * nq);
  if (row >= total_rows) return;
  const int64_t seq0 = (row / S) * S;  // first token of this sequence
  const int i = static_cast<int>(row - seq0);
  const int kh = h / (nq / nkv);
  const uint16_t* qp = q + row * ldq + h * 128 + lane * 4;
  const uint2 qraw = *reinterpret_cast<const uint2*>(qp);
  const float q0 = bf(qraw.x & 0xFFFF), q1 = bf(qraw.x >> 16), q2 = bf(qraw.y & 0xFFFF), q3 = bf(qraw.y >> 16);
  float m = __int_as_float(0xFF800000), l = 0.0f;
  float o0 = 0.0f, o1 = 0.0f, o2 = 0.0f, o3 = 0.0f;
  for (int j = 0; j <= i; ++j) {
    const int64_t kr = seq0 + j;
    const uint2 kraw = *reinterpret_cast<const uint2*>(k + kr * ldk + kh * 128 + lane * 4);
    float part = 0.0f;
    part = __fmaf_rn(q0, bf(kraw.x & 0xFFFF), part);
    part = __fmaf_rn(q1, bf(kraw.x >> 16), part);
    part = __fmaf_rn(q2, bf(kraw.y & 0xFFFF), part);
    part = __fmaf_rn(q3, bf(kraw.y >> 16), part);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) part = __fadd_rn(part, __shfl_xor_sync(0xffffffffu, part, d));
    const float s = __fmul_rn(part, scale);
    const uint2 vraw = *reinterpret_cast<const uint2*>(v + kr * ldv + kh * 128 + lane * 4);
    const float v0 = bf(vraw.x & 0xFFFF), v1 = bf(vraw.x >> 16), v2 = bf(vraw.y & 0xFFFF), v3 = bf(vraw.y >> 16);
    if (s > m) {
      const float a = tb_exp(__fsub_rn(m, s));
      l = __fadd_rn(__fmul_rn(l, a), 1.0f);
      o0 = __fadd_rn(__fmul_rn(o0, a), v0);
      o1 = __fadd_rn(__fmul_rn(o1, a), v1);
      o2 = __fadd_rn(__fmul_rn(o2, a), v2);
      o3 = __fadd_rn(__fmul_rn(o3, a), v3);
      m = s;
    } else {
      const float pj = tb_exp(__fsub_rn(s, m));
      l = __fadd_rn(l, pj);
      o0 = __fmaf_rn(pj, v0, o0);
      o1 = __fmaf_rn(pj, v1, o1);
      o2 = __fmaf_rn(pj, v2, o2);
      o3 = __fmaf_rn(pj, v3, o3);
    }
  }
  uint16_t* op = out + row * ldo + h * 128 + lane * 4;
  const uint32_t lo = static_cast<uint32_t>(f32_to_bf16_bits(__fdiv_rn(o0, l))) |
                      (static_cast<uint32_t>(f32_to_bf16_bits(__fdiv_rn(o1, l))) << 16);
  const uint32_t hi = static_cast<uint32_t>(f32_to_bf16_bits(__fdiv_rn(o2, l))) |
                      (static_cast<uint32_t>(f32_to_bf16_bits(__fdiv_rn(o3, l))) << 16);
  *reinterpret_cast<uint2*>(op) = make_uint2(lo, hi);
}

// ---- SiLU(gate) * up  (demo.cpp:36-45, :171-174) ---------------------------------------
// gu: f32 [M, ld] with gate in columns [0, I) and up in [I, 2I).  silu(z) = z / (1 + exp(-z)).
__global__ void silu_mul_kernel(const float* __restrict__ gu, int64_t ld, int64_t I, uint16_t* __restrict__ out,
                                int64_t ldo) {
  const int64_t row = blockIdx.y;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < I;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float z = gu[row * ld + j];
    const float s = __fdiv_rn(z, __fadd_rn(1.0f, tb_exp(-z)));
    out[row * ldo + j] = f32_to_bf16_bits(__fmul_rn(s, gu[row * ld + I + j]));
  }
}

// ---- residual: h = bf16(h + f)  (demo.cpp:216) -------------------------------------------------
__global__ void residual_kernel(uint16_t* __restrict__ h, int64_t ldh, const float* __restrict__ f, int64_t ldf,
                                int64_t cols) {
  const int64_t row = blockIdx.y;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    h[row * ldh + j] = f32_to_bf16_bits(__fadd_rn(bf(h[row * ldh + j]), f[row * ldf + j]));
}

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
  TBIK_TRY(need_device());
  const int64_t rows = batch * seq_len;
  const int64_t warps = rows * n_q_heads;
  const int64_t blocks = (warps * 32 + 255) / 256;
  attn_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(q), ldq, static_cast<const uint16_t*>(k), ldk, static_cast<const uint16_t*>(v), ldv,
      seq_len, n_q_heads, n_kv_heads, scale, static_cast<uint16_t*>(out), ldo, rows);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_silu_mul(const float* gate_up, int64_t ld, int64_t rows, int64_t inter, void* out, int64_t ldo,
                          void* stream) {
  if (!gate_up || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || inter < 1 || rows > 65535) return set_error(TBIK_BAD_DIMENSION, "silu_mul: bad dimensions");
  TBIK_TRY(need_device());
  silu_mul_kernel<<<row_grid(rows, inter, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      gate_up, ld, inter, static_cast<uint16_t*>(out), ldo);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_residual_add(void* h, int64_t ldh, const float* f, int64_t ldf, int64_t rows, int64_t cols,
                              void* stream) {
  if (!h || !f) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || cols < 1 || rows > 65535) return set_error(TBIK_BAD_DIMENSION, "residual: bad dimensions");
  TBIK_TRY(need_device());
  residual_kernel<<<row_grid(rows, cols, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint16_t*>(h), ldh, f, ldf, cols);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

}  // extern "C"
