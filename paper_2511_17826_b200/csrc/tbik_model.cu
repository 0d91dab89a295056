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

// tbik_attn_tc5.cu
tbik_status launch_attn_tc5(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                            int64_t batch, int S, int nq, int nkv, float scale_log2, void* out, int64_t ldo,
                            cudaStream_t s);

namespace {

__device__ __forceinline__ float bf(uint16_t b) { return bf16_bits_to_f32(b); }

// ---- embedding gather -------------------------------------------------------------
__global__ void embed_kernel(const uint16_t* __restrict__ table, int64_t H, const int64_t* __restrict__ ids,
                             int64_t V, uint16_t* __restrict__ out, int* __restrict__ bad) {
  pdl_wait();
  pdl_trigger();
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
  pdl_trigger();
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

// One quad of a head: out[d..d+3] and out[d+half..+3] from x[d..], x[d+half..] --
// rope_kernel's operations, four lanes at a time.
__device__ __forceinline__ void rope_quad(const float* xh, int d, int half, const float* cs, const float* sn_t,
                                          uint16_t* o) {
  const float4 a = *reinterpret_cast<const float4*>(xh + d);
  const float4 b = *reinterpret_cast<const float4*>(xh + d + half);
  const float4 c = *reinterpret_cast<const float4*>(cs + d);
  const float4 sn = *reinterpret_cast<const float4*>(sn_t + d);
  const float lo0 = __fsub_rn(__fmul_rn(a.x, c.x), __fmul_rn(b.x, sn.x));
  const float lo1 = __fsub_rn(__fmul_rn(a.y, c.y), __fmul_rn(b.y, sn.y));
  const float lo2 = __fsub_rn(__fmul_rn(a.z, c.z), __fmul_rn(b.z, sn.z));
  const float lo3 = __fsub_rn(__fmul_rn(a.w, c.w), __fmul_rn(b.w, sn.w));
  const float hi0 = __fadd_rn(__fmul_rn(b.x, c.x), __fmul_rn(a.x, sn.x));
  const float hi1 = __fadd_rn(__fmul_rn(b.y, c.y), __fmul_rn(a.y, sn.y));
  const float hi2 = __fadd_rn(__fmul_rn(b.z, c.z), __fmul_rn(a.z, sn.z));
  const float hi3 = __fadd_rn(__fmul_rn(b.w, c.w), __fmul_rn(a.w, sn.w));
  *reinterpret_cast<uint2*>(o + d) =
      make_uint2(f32_to_bf16_bits(lo0) | (static_cast<uint32_t>(f32_to_bf16_bits(lo1)) << 16),
                 f32_to_bf16_bits(lo2) | (static_cast<uint32_t>(f32_to_bf16_bits(lo3)) << 16));
  *reinterpret_cast<uint2*>(o + d + half) =
      make_uint2(f32_to_bf16_bits(hi0) | (static_cast<uint32_t>(f32_to_bf16_bits(hi1)) << 16),
                 f32_to_bf16_bits(hi2) | (static_cast<uint32_t>(f32_to_bf16_bits(hi3)) << 16));
}

// Vectorised form (D % 8 == 0, 16-byte aligned rows): thread = (head, 4 dims d..d+3
// of the first half); it produces out[d..d+3] and out[d+D/2..+3] with the same
// operations as rope_kernel.  Several rows per CTA (blockDim.y).
__global__ void rope_vec_kernel(const float* __restrict__ x, int64_t ldx, int64_t col0, int heads, int D,
                                const int* __restrict__ pos, const float* __restrict__ cos_t,
                                const float* __restrict__ sin_t, uint16_t* __restrict__ out, int64_t ldo,
                                int64_t rows) {
  pdl_wait();
  pdl_trigger();
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.y + threadIdx.y;
  if (row >= rows) return;
  const int half = D / 2, qpr = half / 4;  // float4 quads per half head
  const int p = pos[row];
  for (int e = threadIdx.x; e < heads * qpr; e += blockDim.x) {
    const int h = e / qpr, d = (e - h * qpr) * 4;
    const float* xh = x + row * ldx + col0 + h * D;
    rope_quad(xh, d, half, cos_t + static_cast<int64_t>(p) * half, sin_t + static_cast<int64_t>(p) * half,
              out + row * ldo + h * D);
  }
}

// f32 -> bf16 copy of a column block (V of qkv, storage casts).
__global__ void cast_kernel(const float* __restrict__ x, int64_t ldx, int64_t cols, uint16_t* __restrict__ out,
                            int64_t ldo) {
  pdl_wait();
  pdl_trigger();
  const int64_t row = blockIdx.y;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[row * ldo + j] = f32_to_bf16_bits(x[row * ldx + j]);
}

// The attention inputs from one f32 qkv row in ONE launch: RoPE of the nq q heads
// (columns [0, nq D)) and the nkv k heads (the next nkv D columns) and the bf16
// cast of v (the last nkv D) -- rope_vec_kernel's and cast_kernel's operations per
// element, three launches folded into one (D % 8 == 0, 16-byte aligned rows).
__global__ void rope_qkv_kernel(const float* __restrict__ x, int64_t ldx, int nq, int nkv, int D,
                                const int* __restrict__ pos, const float* __restrict__ cos_t,
                                const float* __restrict__ sin_t, uint16_t* __restrict__ q_out,
                                uint16_t* __restrict__ k_out, uint16_t* __restrict__ v_out, int64_t rows) {
  pdl_wait();
  pdl_trigger();
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.y + threadIdx.y;
  if (row >= rows) return;
  const int half = D / 2, qpr = half / 4;
  const int p = pos[row];
  const float* xr = x + row * ldx;
  const float* cs = cos_t + static_cast<int64_t>(p) * half;
  const float* sn = sin_t + static_cast<int64_t>(p) * half;
  const int nrope = (nq + nkv) * qpr, nv = nkv * D / 4;
  for (int e = threadIdx.x; e < nrope + nv; e += blockDim.x) {
    if (e < nrope) {
      const int h = e / qpr, d = (e - h * qpr) * 4;
      if (h < nq)
        rope_quad(xr + h * D, d, half, cs, sn, q_out + row * nq * D + h * D);
      else
        rope_quad(xr + h * D, d, half, cs, sn, k_out + row * nkv * D + (h - nq) * D);
    } else {
      const int j = (e - nrope) * 4;
      const float4 f = *reinterpret_cast<const float4*>(xr + (nq + nkv) * D + j);
      *reinterpret_cast<uint2*>(v_out + row * nkv * D + j) =
          make_uint2(f32_to_bf16_bits(f.x) | (static_cast<uint32_t>(f32_to_bf16_bits(f.y)) << 16),
                     f32_to_bf16_bits(f.z) | (static_cast<uint32_t>(f32_to_bf16_bits(f.w)) << 16));
    }
  }
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
  pdl_wait();
  pdl_trigger();
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

// ---- causal GQA prefill attention, tensor-core flash form ------------------------------------
// The fast attention of the tcgen05-leaf forward.  Deterministic and batch / head-
// sharding invariant by construction, but NOT the exact two-pass order above (its
// dot products run on mma.sync tensor cores): parity against attn2 / the oracle is
// a tolerance, bit identity across TP and batch is exact.  Canonical form, per
// (sequence, q head, query i) with keys in blocks of 64 from key 0:
//   per block: s = q.k (mma.sync m16n8k16 bf16 -> f32), masked keys -inf
//              m' = max(m, rowmax s)   (quad shuffles xor 1, 2)
//              p  = exp2(s c - m' c), c = scale * log2 e;  alpha = exp2(m c - m' c)
//              l  = l alpha + (sequential sum of the lane's p);  O = O alpha + bf16(p) . v
//   out = bf16(O / (quad sum of l))
// One CTA = (64-query block, q head, sequence), 4 warps x 16 query rows; K and V
// blocks double-buffered in shared memory by cp.async, B fragments by ldmatrix
// (.trans for V).
constexpr int FQ = 64;          // queries per CTA
constexpr int FK = 64;          // keys per block
constexpr int FKP = AD + 8;     // padded bf16 row of a staged K / V block (272 B: conflict-free ldmatrix)
constexpr int FSTAGE = FK * FKP;  // elements per staged block

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  return static_cast<uint32_t>(f32_to_bf16_bits(lo)) | (static_cast<uint32_t>(f32_to_bf16_bits(hi)) << 16);
}

// SV1: the V block single-buffered (K double-buffered): 3 staged blocks = 52 KB,
// four CTAs per SM instead of three; V(kb) is loaded while Q.K(kb) and the
// softmax run.  Same MMAs in the same order either way.
template <bool SV1>
__global__ void __launch_bounds__(128) attn_mma_kernel(const uint16_t* __restrict__ q, int64_t ldq,
                                                       const uint16_t* __restrict__ k, int64_t ldk,
                                                       const uint16_t* __restrict__ v, int64_t ldv, int S, int nq,
                                                       int nkv, float scale_log2, uint16_t* __restrict__ out,
                                                       int64_t ldo) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint16_t fsm[];  // [2 buffers][K block, V block] (SV1: K0, K1, V)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int qb = static_cast<int>(gridDim.z) - 1 - static_cast<int>(blockIdx.z), h = blockIdx.x;
  const int64_t seq0 = static_cast<int64_t>(blockIdx.y) * S;
  const int kh = h / (nq / nkv);
  const int r0 = qb * FQ + warp * 16 + g;  // this thread's rows r0 and r0 + 8
  const int last_key = min(S, (qb + 1) * FQ) - 1;
  const int nkb = last_key / FK + 1;

  auto kbuf = [&](int buf) { return SV1 ? fsm + buf * FSTAGE : fsm + buf * 2 * FSTAGE; };
  auto vbuf = [&](int buf) { return SV1 ? fsm + 2 * FSTAGE : fsm + buf * 2 * FSTAGE + FSTAGE; };
  // keys past the causal end / sequence as zeros
  auto stage_part = [&](int kb, uint16_t* dst, const uint16_t* src, int64_t ld) {
#pragma unroll
    for (int x = 0; x < FK * AD / 8 / 128; ++x) {
      const int e = tid + x * 128;
      const int r = e / (AD / 8), c = (e % (AD / 8)) * 8;
      const int key = kb * FK + r;
      const bool ok = key <= last_key;
      const int64_t row = seq0 + (ok ? key : 0);
      cp_async16(dst + r * FKP + c, src + row * ld + kh * AD + c, ok);
    }
  };
  auto stage = [&](int kb, int buf) {
    stage_part(kb, kbuf(buf), k, ldk);
    stage_part(kb, vbuf(buf), v, ldv);
    cp_async_commit();
  };
  if constexpr (SV1) {
    stage_part(0, kbuf(0), k, ldk);
    cp_async_commit();
    stage_part(0, vbuf(0), v, ldv);
    cp_async_commit();
  } else {
    stage(0, 0);
  }

  // Q fragments (16 rows x 128 d per warp): qa[kstep][4]
  uint32_t qa[AD / 16][4];
  {
    const int ra = min(r0, S - 1), rb = min(r0 + 8, S - 1);
    const uint16_t* qpa = q + (seq0 + ra) * ldq + h * AD;
    const uint16_t* qpb = q + (seq0 + rb) * ldq + h * AD;
#pragma unroll
    for (int ks = 0; ks < AD / 16; ++ks) {
      qa[ks][0] = *reinterpret_cast<const uint32_t*>(qpa + ks * 16 + 2 * t);
      qa[ks][1] = *reinterpret_cast<const uint32_t*>(qpb + ks * 16 + 2 * t);
      qa[ks][2] = *reinterpret_cast<const uint32_t*>(qpa + ks * 16 + 2 * t + 8);
      qa[ks][3] = *reinterpret_cast<const uint32_t*>(qpb + ks * 16 + 2 * t + 8);
    }
  }
  float o[AD / 8][4];
#pragma unroll
  for (int n = 0; n < AD / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.0f;
  const float NEG_INF = __int_as_float(0xFF800000);
  float m[2] = {NEG_INF, NEG_INF}, l[2] = {0.0f, 0.0f};
  // ldmatrix row addresses: lane i feeds row i % 8 of matrix i / 8
  const int lr = lane & 7, lm = lane >> 3;

  for (int kb = 0; kb < nkb; ++kb) {
    if constexpr (SV1) {
      // pending: V(kb) [, K(kb + 1) issued now]; K(kb) is complete after the wait
      if (kb + 1 < nkb) {
        stage_part(kb + 1, kbuf((kb + 1) & 1), k, ldk);
        cp_async_commit();
        cp_async_wait<2>();
      } else {
        cp_async_wait<1>();
      }
    } else if (kb + 1 < nkb) {
      stage(kb + 1, (kb + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint16_t* sK = kbuf(kb & 1);
    const uint16_t* sV = vbuf(kb & 1);
    // s = q . k for this warp's 16 rows x 64 keys (8 n-tiles of 8 keys).  ldmatrix x4
    // matrices: (keys n*8.., d ks*16 + 0/8) for n-tile pair (n, n+1)
    float sc[FK / 8][4];
#pragma unroll
    for (int n = 0; n < FK / 8; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.0f;
#pragma unroll
    for (int ks = 0; ks < AD / 16; ++ks) {
#pragma unroll
      for (int n = 0; n < FK / 8; n += 2) {
        uint32_t b[4];  // b0(n), b1(n), b0(n+1), b1(n+1)
        ldsm_x4(b, sK + ((n + (lm >> 1)) * 8 + lr) * FKP + ks * 16 + (lm & 1) * 8);
        mma_bf16_16816(sc[n], qa[ks], b[0], b[1]);
        mma_bf16_16816(sc[n + 1], qa[ks], b[2], b[3]);
      }
    }
    // causal / sequence mask, block row max
    float bm[2] = {NEG_INF, NEG_INF};
#pragma unroll
    for (int n = 0; n < FK / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * FK + n * 8 + 2 * t + (e & 1);
        const int row = r0 + (e >> 1) * 8;
        if (key > row || key > last_key) sc[n][e] = NEG_INF;
        bm[e >> 1] = fmaxf(bm[e >> 1], sc[n][e]);
      }
    float alpha[2], mc[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      bm[x] = fmaxf(bm[x], __shfl_xor_sync(0xffffffffu, bm[x], 1));
      bm[x] = fmaxf(bm[x], __shfl_xor_sync(0xffffffffu, bm[x], 2));
      const float mn = fmaxf(m[x], bm[x]);
      // rows whose keys are all masked so far (only rows past the sequence end) keep m = -inf
      mc[x] = mn == NEG_INF ? 0.0f : __fmul_rn(mn, scale_log2);
      alpha[x] = m[x] == NEG_INF ? 0.0f : exp2f(__fsub_rn(__fmul_rn(m[x], scale_log2), mc[x]));
      m[x] = mn;
    }
    // p = exp2(s c - m c); l = l alpha + sum p; P packed as the A operand of P.V
    uint32_t pa[FK / 16][4];
    float ps[2] = {0.0f, 0.0f};
#pragma unroll
    for (int n = 0; n < FK / 8; ++n) {
      float pv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        pv[e] = exp2f(__fsub_rn(__fmul_rn(sc[n][e], scale_log2), mc[e >> 1]));
        ps[e >> 1] = __fadd_rn(ps[e >> 1], pv[e]);
      }
      pa[n >> 1][(n & 1) * 2 + 0] = pack_bf16x2(pv[0], pv[1]);
      pa[n >> 1][(n & 1) * 2 + 1] = pack_bf16x2(pv[2], pv[3]);
    }
#pragma unroll
    for (int x = 0; x < 2; ++x) l[x] = __fadd_rn(__fmul_rn(l[x], alpha[x]), ps[x]);
#pragma unroll
    for (int n = 0; n < AD / 8; ++n) {
      o[n][0] = __fmul_rn(o[n][0], alpha[0]);
      o[n][1] = __fmul_rn(o[n][1], alpha[0]);
      o[n][2] = __fmul_rn(o[n][2], alpha[1]);
      o[n][3] = __fmul_rn(o[n][3], alpha[1]);
    }
    if constexpr (SV1) {  // V(kb) complete (only K(kb + 1) may still be in flight)
      if (kb + 1 < nkb)
        cp_async_wait<1>();
      else
        cp_async_wait<0>();
      __syncthreads();
    }
    // O += P . V: B fragments of V [key][d] by ldmatrix.trans, matrices (keys ks*16 +
    // 0/8, d n*8..) for d-tile pair (n, n+1)
#pragma unroll
    for (int ks = 0; ks < FK / 16; ++ks) {
#pragma unroll
      for (int n = 0; n < AD / 8; n += 2) {
        uint32_t b[4];
        ldsm_x4_t(b, sV + (ks * 16 + (lm & 1) * 8 + lr) * FKP + (n + (lm >> 1)) * 8);
        mma_bf16_16816(o[n], pa[ks], b[0], b[1]);
        mma_bf16_16816(o[n + 1], pa[ks], b[2], b[3]);
      }
    }
    __syncthreads();  // this buffer is restaged two blocks later (SV1: V now)
    if constexpr (SV1) {
      if (kb + 1 < nkb) {
        stage_part(kb + 1, vbuf(0), v, ldv);
        cp_async_commit();
      }
    }
  }
  // l over the quad (xor 1 then xor 2), out = bf16(O / l)
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    l[x] = __fadd_rn(l[x], __shfl_xor_sync(0xffffffffu, l[x], 1));
    l[x] = __fadd_rn(l[x], __shfl_xor_sync(0xffffffffu, l[x], 2));
  }
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    const int row = r0 + 8 * x;
    if (row >= S) continue;
    uint16_t* op = out + (seq0 + row) * ldo + h * AD + 2 * t;
#pragma unroll
    for (int n = 0; n < AD / 8; ++n)
      *reinterpret_cast<uint32_t*>(op + n * 8) =
          pack_bf16x2(__fdiv_rn(o[n][2 * x], l[x]), __fdiv_rn(o[n][2 * x + 1], l[x]));
  }
}

// ---- SiLU(gate) * up  (demo.cpp:36-45, :171-174) ---------------------------------------
// gu: f32 [M, ld] with gate in columns [0, I) and up in [I, 2I).  silu(z) = z / (1 + exp(-z)).
__device__ __forceinline__ uint16_t silu_mul1(float z, float up) { return tb_silu_mul_bf16(z, up); }

// Interleaved layout (gate_j at column 2j, up_j at 2j+1), the fallback of the
// fused gate_up GEMM (tbik_tree_matmul_silu_mul) when its epilogue cannot run.
__global__ void silu_mul_il_kernel(const float* __restrict__ gu, int64_t ld, int64_t I, uint16_t* __restrict__ out,
                                   int64_t ldo) {
  pdl_trigger();
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
  pdl_trigger();
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
  pdl_trigger();
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
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int* bad = static_cast<int*>(workspace(16, 3, s));
  if (!bad) return set_error(TBIK_CUDA_ERROR, "workspace");
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
  const bool vec = head_dim % 8 == 0 && ldx % 4 == 0 && col0 % 4 == 0 && ldo % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 7) == 0 &&
                   (reinterpret_cast<uintptr_t>(cos_table) & 15) == 0 && (reinterpret_cast<uintptr_t>(sin_table) & 15) == 0;
  if (vec) {
    const int threads = heads * head_dim / 8;
    const int tx = threads < 256 ? ((threads + 31) / 32) * 32 : 256;
    const int ty = 256 / tx;
    TBIK_CUDA(launch_pdl(rope_vec_kernel, dim3(static_cast<unsigned>((rows + ty - 1) / ty)), dim3(tx, ty), 0,
                         static_cast<cudaStream_t>(stream), x, ldx, col0, heads, head_dim, positions, cos_table,
                         sin_table, static_cast<uint16_t*>(out), ldo, rows));
  } else {
    rope_kernel<<<static_cast<unsigned>(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x, ldx, col0, heads, head_dim, positions, cos_table, sin_table, static_cast<uint16_t*>(out), ldo);
  }
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_rope_qkv(const float* qkv, int64_t ld, int n_q_heads, int n_kv_heads, int head_dim,
                          const int* positions, const float* cos_table, const float* sin_table, void* q_out,
                          void* k_out, void* v_out, int64_t rows, void* stream) {
  if (!qkv || !positions || !cos_table || !sin_table || !q_out || !k_out || !v_out)
    return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (head_dim % 8 || n_q_heads < 1 || n_kv_heads < 1 || rows < 1)
    return set_error(TBIK_BAD_DIMENSION, "rope_qkv: bad dimensions");
  const auto a16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  if (ld % 4 || !a16(qkv) || !a16(cos_table) || !a16(sin_table) || (reinterpret_cast<uintptr_t>(q_out) & 7) ||
      (reinterpret_cast<uintptr_t>(k_out) & 7) || (reinterpret_cast<uintptr_t>(v_out) & 7))
    return set_error(TBIK_BAD_ARGUMENT, "rope_qkv: 16-byte aligned f32 rows and 8-byte aligned outputs required");
  TBIK_TRY(need_device());
  const int rows_per_cta = 2;
  TBIK_CUDA(launch_pdl(rope_qkv_kernel, dim3(static_cast<unsigned>((rows + rows_per_cta - 1) / rows_per_cta)),
                       dim3(256, rows_per_cta), 0, static_cast<cudaStream_t>(stream), qkv, ld, n_q_heads, n_kv_heads,
                       head_dim, positions, cos_table, sin_table, static_cast<uint16_t*>(q_out),
                       static_cast<uint16_t*>(k_out), static_cast<uint16_t*>(v_out), rows));
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_cast_bf16(const float* x, int64_t ldx, int64_t rows, int64_t cols, void* out, int64_t ldo,
                           void* stream) {
  if (!x || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1 || cols < 1 || rows > 65535) return set_error(TBIK_BAD_DIMENSION, "cast: bad dimensions");
  TBIK_TRY(need_device());
  TBIK_CUDA(launch_pdl(cast_kernel, row_grid(rows, cols, 256), dim3(256), 0, static_cast<cudaStream_t>(stream), x, ldx,
                       cols, static_cast<uint16_t*>(out), ldo));
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
  // per launch: the attribute is per device context
  TBIK_CUDA(cudaFuncSetAttribute(attn2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  dim3 grid(static_cast<unsigned>(n_q_heads), static_cast<unsigned>(batch),
            static_cast<unsigned>((seq_len + AQ - 1) / AQ));
  TBIK_CUDA(launch_pdl(attn2_kernel, grid, dim3(4 * AQ), smem, static_cast<cudaStream_t>(stream),
                       static_cast<const uint16_t*>(q), ldq, static_cast<const uint16_t*>(k), ldk,
                       static_cast<const uint16_t*>(v), ldv, seq_len, n_q_heads, n_kv_heads, scale,
                       static_cast<uint16_t*>(out), ldo));
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

tbik_status tbik_attention_prefill_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                                      int64_t ldv, int64_t batch, int seq_len, int n_q_heads, int n_kv_heads,
                                      int head_dim, float scale, void* out, int64_t ldo, void* stream) {
  if (!q || !k || !v || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (head_dim != 128) return set_error(TBIK_UNSUPPORTED, "attention: head_dim must be 128");
  if (n_kv_heads < 1 || n_q_heads % n_kv_heads) return set_error(TBIK_BAD_DIMENSION, "attention: bad GQA heads");
  if (seq_len < 1 || seq_len > (1 << 20)) return set_error(TBIK_UNSUPPORTED, "attention: seq_len out of range");
  if (batch < 1 || batch > 65535 || n_q_heads > 65535) return set_error(TBIK_BAD_DIMENSION, "attention: grid");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
       reinterpret_cast<uintptr_t>(out)) & 15 || ldq % 8 || ldk % 8 || ldv % 8 || ldo % 8)
    return set_error(TBIK_BAD_ARGUMENT, "attention: 16-byte aligned rows required");
  TBIK_TRY(need_device());
  const float scale_log2 = scale * 1.4426950408889634f;
  dim3 grid(static_cast<unsigned>(n_q_heads), static_cast<unsigned>(batch),
            static_cast<unsigned>((seq_len + FQ - 1) / FQ));
  if (knob(KNOB_ATTN_TC5, 1) != 0)  // tcgen05 form (tbik_attn_tc5.cu, default): its own bits, same tolerance
    return launch_attn_tc5(q, ldq, k, ldk, v, ldv, batch, seq_len, n_q_heads, n_kv_heads, scale_log2, out, ldo,
                           static_cast<cudaStream_t>(stream));
  const bool sv1 = knob(KNOB_ATTN_SV1, 1) != 0;
  const size_t fsmem = (sv1 ? 3 : 4) * FSTAGE * sizeof(uint16_t);
  const auto kern = sv1 ? attn_mma_kernel<true> : attn_mma_kernel<false>;
  TBIK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fsmem)));
  TBIK_CUDA(launch_pdl(kern, grid, dim3(128), fsmem, static_cast<cudaStream_t>(stream),
                       static_cast<const uint16_t*>(q), ldq, static_cast<const uint16_t*>(k), ldk,
                       static_cast<const uint16_t*>(v), ldv, seq_len, n_q_heads, n_kv_heads, scale_log2,
                       static_cast<uint16_t*>(out), ldo));
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
