// tbik_mathfn.cuh -- the shared, explicitly-rounded exp / log used by every
// kernel that needs a transcendental (log-softmax, SiLU, attention).  The exact
// same operation sequence is restated on the CPU in oracle/tbik_oracle.c
// (tbo_exp / tbo_log), so GPU and oracle agree bit for bit; glibc and CUDA expf /
// logf do not.
#pragma once

#include "tbik_common.cuh"

namespace tbik_b200 {

__device__ __forceinline__ float tb_exp(float x) {
  if (x != x) return x;
  if (x < -103.0f) return 0.0f;
  if (x > 88.5f) return __int_as_float(0x7F800000);
  const float magic = 12582912.0f;
  const float t = __fmaf_rn(x, 1.44269502162933349609f, magic);
  const float kf = __fsub_rn(t, magic);
  float r = __fmaf_rn(kf, -0.693359375f, x);
  r = __fmaf_rn(kf, 2.12194440e-4f, r);
  float p = 1.9875691500e-4f;
  p = __fmaf_rn(p, r, 1.3981999507e-3f);
  p = __fmaf_rn(p, r, 8.3334519073e-3f);
  p = __fmaf_rn(p, r, 4.1665795894e-2f);
  p = __fmaf_rn(p, r, 1.6666665459e-1f);
  p = __fmaf_rn(p, r, 5.0000001201e-1f);
  const float r2 = __fmul_rn(r, r);
  float y = __fmaf_rn(p, r2, r);
  y = __fadd_rn(y, 1.0f);
  int k = static_cast<int>(kf);
  if (k < -125) {
    y = __fmul_rn(y, __uint_as_float(static_cast<uint32_t>(127 - 64) << 23));
    k += 64;
  }
  return __fmul_rn(y, __uint_as_float(static_cast<uint32_t>(k + 127) << 23));
}

// tb_exp for x in [-inf, 0] (no NaN): the same operation sequence as tb_exp, so
// the same bits, with the branches turned into selects and the exponent taken
// from the magic-number sum (t = magic + kf exactly, |kf| < 2^22) instead of a
// float->int conversion.  Used on the log-softmax hot loop (x - max <= 0).
__device__ __forceinline__ float tb_exp_nonpos(float x) {
  const float magic = 12582912.0f;  // 0x4B400000
  const float t = __fmaf_rn(x, 1.44269502162933349609f, magic);
  const float kf = __fsub_rn(t, magic);
  float r = __fmaf_rn(kf, -0.693359375f, x);
  r = __fmaf_rn(kf, 2.12194440e-4f, r);
  float p = 1.9875691500e-4f;
  p = __fmaf_rn(p, r, 1.3981999507e-3f);
  p = __fmaf_rn(p, r, 8.3334519073e-3f);
  p = __fmaf_rn(p, r, 4.1665795894e-2f);
  p = __fmaf_rn(p, r, 1.6666665459e-1f);
  p = __fmaf_rn(p, r, 5.0000001201e-1f);
  const float r2 = __fmul_rn(r, r);
  float y = __fmaf_rn(p, r2, r);
  y = __fadd_rn(y, 1.0f);
  // k = t_bits - magic_bits; 2^k has bits (k + 127) << 23 = (t_bits << 23) + C (mod 2^32)
  const uint32_t tb = __float_as_uint(t);
  const bool tiny = kf < -125.0f;
  y = __fmul_rn(y, tiny ? __uint_as_float(static_cast<uint32_t>(127 - 64) << 23) : 1.0f);  // *1 is exact
  const uint32_t sc = (tb << 23) + ((127u - 0x4B400000u) << 23) + (tiny ? (64u << 23) : 0u);
  const float res = __fmul_rn(y, __uint_as_float(sc));
  return x < -103.0f ? 0.0f : res;
}

// tb_exp_nonpos for x >= -86 (then k >= -124: no gradual-underflow scaling and
// no flush to zero apply), bit-identical to it on that range and for NaN.  The
// caller proves the range for a whole block of arguments first.
__device__ __forceinline__ float tb_exp_nonpos_normal(float x) {
  const float magic = 12582912.0f;
  const float t = __fmaf_rn(x, 1.44269502162933349609f, magic);
  const float kf = __fsub_rn(t, magic);
  float r = __fmaf_rn(kf, -0.693359375f, x);
  r = __fmaf_rn(kf, 2.12194440e-4f, r);
  float p = 1.9875691500e-4f;
  p = __fmaf_rn(p, r, 1.3981999507e-3f);
  p = __fmaf_rn(p, r, 8.3334519073e-3f);
  p = __fmaf_rn(p, r, 4.1665795894e-2f);
  p = __fmaf_rn(p, r, 1.6666665459e-1f);
  p = __fmaf_rn(p, r, 5.0000001201e-1f);
  const float r2 = __fmul_rn(r, r);
  float y = __fmaf_rn(p, r2, r);
  y = __fadd_rn(y, 1.0f);
  const uint32_t sc = (__float_as_uint(t) << 23) + ((127u - 0x4B400000u) << 23);
  return __fmul_rn(y, __uint_as_float(sc));
}

// Packed two-lane f32 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2): each lane is
// the IEEE RN operation of the scalar form, so results are bit-identical and the
// instruction count of a polynomial halves.
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b,
                                                     unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// tb_exp_nonpos_normal of two arguments at once (x in [-86, 0] or NaN), same bits.
__device__ __forceinline__ void tb_exp_nonpos_normal2(float a, float b, float& ea, float& eb) {
  const unsigned long long magic = f2_pack(12582912.0f, 12582912.0f);
  const unsigned long long x = f2_pack(a, b);
  const unsigned long long t = f2_fma(x, f2_pack(1.44269502162933349609f, 1.44269502162933349609f), magic);
  const unsigned long long kf = f2_sub(t, magic);
  unsigned long long r = f2_fma(kf, f2_pack(-0.693359375f, -0.693359375f), x);
  r = f2_fma(kf, f2_pack(2.12194440e-4f, 2.12194440e-4f), r);
  unsigned long long p = f2_fma(f2_pack(1.9875691500e-4f, 1.9875691500e-4f), r,
                                f2_pack(1.3981999507e-3f, 1.3981999507e-3f));
  p = f2_fma(p, r, f2_pack(8.3334519073e-3f, 8.3334519073e-3f));
  p = f2_fma(p, r, f2_pack(4.1665795894e-2f, 4.1665795894e-2f));
  p = f2_fma(p, r, f2_pack(1.6666665459e-1f, 1.6666665459e-1f));
  p = f2_fma(p, r, f2_pack(5.0000001201e-1f, 5.0000001201e-1f));
  const unsigned long long r2 = f2_mul(r, r);
  unsigned long long y = f2_fma(p, r2, r);
  y = f2_add(y, f2_pack(1.0f, 1.0f));
  float tl, th;
  f2_unpack(t, tl, th);
  const uint32_t sl = (__float_as_uint(tl) << 23) + ((127u - 0x4B400000u) << 23);
  const uint32_t sh = (__float_as_uint(th) << 23) + ((127u - 0x4B400000u) << 23);
  f2_unpack(f2_mul(y, f2_pack(__uint_as_float(sl), __uint_as_float(sh))), ea, eb);
}

// (m, s) state of one 16-logit log-softmax chunk held in registers (the canonical
// chunk of tbo_tree_logsoftmax): m = sequential max (x > m ? x : m) from v[0],
// s = ((0 + e_0) + e_1) + ... + e_15, e_i = exp(x_i - m) in ascending order;
// all -inf -> (-inf, 0).  Shared by the log-softmax kernels and the lm_head GEMM
// epilogue so both produce the same bits.
constexpr int TB_MS_CHUNK = 16;
__device__ __forceinline__ void tb_ms_chunk16(const float (&v)[TB_MS_CHUNK], float& m_out, float& s_out) {
  const float NEG_INF = __int_as_float(0xFF800000);
  // fmaxf gives the sequential compare's bits unless the maximum is a zero (only
  // its sign is ambiguous): redo those in order (NaN is outside the contract).
  float m = v[0], lo = v[0];
#pragma unroll
  for (int k = 1; k < TB_MS_CHUNK; ++k) {
    m = fmaxf(m, v[k]);
    lo = fminf(lo, v[k]);
  }
  if (m == 0.0f) {
    m = v[0];
#pragma unroll
    for (int k = 1; k < TB_MS_CHUNK; ++k) m = v[k] > m ? v[k] : m;
  }
  float sum = 0.0f;
  if (m != NEG_INF) {
    // every x - m >= lo - m (rounding is monotone): when that is >= -86 no element
    // needs tb_exp_nonpos's underflow handling -> the packed two-lane polynomial
    if (__fsub_rn(lo, m) >= -86.0f) {
      const unsigned long long m2 = f2_pack(m, m);
#pragma unroll
      for (int k = 0; k < TB_MS_CHUNK; k += 2) {
        float d0, d1, e0, e1;
        f2_unpack(f2_sub(f2_pack(v[k], v[k + 1]), m2), d0, d1);
        tb_exp_nonpos_normal2(d0, d1, e0, e1);
        sum = __fadd_rn(__fadd_rn(sum, e0), e1);
      }
    } else {
#pragma unroll
      for (int k = 0; k < TB_MS_CHUNK; ++k) sum = __fadd_rn(sum, tb_exp_nonpos(__fsub_rn(v[k], m)));
    }
  }
  m_out = m;
  s_out = m == NEG_INF ? 0.0f : sum;
}

// bf16(silu(z) * up), silu(z) = z / (1 + exp(-z))  (demo.cpp:36-45, :171-174) -- the
// one definition used by the SiLU*up kernel and the gate_up GEMM epilogue.
__device__ __forceinline__ uint16_t tb_silu_mul_bf16(float z, float up) {
  const float sl = __fdiv_rn(z, __fadd_rn(1.0f, tb_exp(-z)));
  const float r = __fmul_rn(sl, up);
  const uint32_t u = __float_as_uint(r);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu) != 0) return 0x7FC0;
  return static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

__device__ __forceinline__ float tb_log(float x) {
  if (!(x > 0.0f)) return x == 0.0f ? __int_as_float(0xFF800000) : __int_as_float(0x7FC00000);
  if (x == __int_as_float(0x7F800000)) return x;
  uint32_t u = __float_as_uint(x);
  int e = 0;
  if ((u & 0x7F800000u) == 0) {
    x = __fmul_rn(x, 4294967296.0f);
    u = __float_as_uint(x);
    e = -32;
  }
  e += static_cast<int>((u >> 23) & 0xFF) - 127;
  float m = __uint_as_float((u & 0x007FFFFFu) | 0x3F800000u);
  if (m > 1.41421356237309504880f) {
    m = __fmul_rn(m, 0.5f);
    e += 1;
  }
  const float xm = __fsub_rn(m, 1.0f);
  const float z = __fmul_rn(xm, xm);
  float p = 7.0376836292e-2f;
  p = __fmaf_rn(p, xm, -1.1514610310e-1f);
  p = __fmaf_rn(p, xm, 1.1676998740e-1f);
  p = __fmaf_rn(p, xm, -1.2420140846e-1f);
  p = __fmaf_rn(p, xm, 1.4249322787e-1f);
  p = __fmaf_rn(p, xm, -1.6668057665e-1f);
  p = __fmaf_rn(p, xm, 2.0000714765e-1f);
  p = __fmaf_rn(p, xm, -2.4999993993e-1f);
  p = __fmaf_rn(p, xm, 3.3333331174e-1f);
  float y = __fmul_rn(p, xm);
  y = __fmul_rn(y, z);
  const float fe = static_cast<float>(e);
  y = __fmaf_rn(fe, -2.12194440e-4f, y);
  y = __fmaf_rn(z, -0.5f, y);
  float r = __fadd_rn(xm, y);
  r = __fmaf_rn(fe, 0.693359375f, r);
  return r;
}

}  // namespace tbik_b200
