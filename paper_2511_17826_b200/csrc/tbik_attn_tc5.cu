// tbik_attn_tc5.cu -- causal GQA prefill attention on tcgen05 (schedule knob attn_tc5).
//
// The tensor-core flash form of tbik_attention_prefill_tc (tbik_model.cu), re-laid for
// the 5th-generation tensor cores: one CTA = 128 queries of one (sequence, q head),
// key blocks of 128.  Per block j:
//   S   = Q . K_j^T            tcgen05.mma M=128 N=128 K=128 (8 x K=16), S in TMEM
//   row = thread (TMEM lane): causal mask, m' = max(m, max_j s), alpha = exp2((m - m') c),
//         p = exp2(s c - m' c), l = l alpha + (p_0 + p_1 + ...) in key order, P = bf16(p)
//   O   = alpha O (rows whose max moved; O in TMEM, read and written back by its row's
//         thread), then O += P . V_j (8 x K=16; P from shared memory, V MN-major)
// and out = bf16(O / l).  Every row is computed by one thread in a fixed order from
// the same operands whatever the batch composition or head sharding, so the bits
// are batch- and TP-invariant; they differ from the mma.sync form's (64-key blocks,
// quad-split row sums), within the same tolerance of the exact two-pass kernel.
// Q, K_j, V_j arrive by TMA through 3-D maps {d, position, sequence}: keys past the
// sequence end read as zeros.  Q 32 KB + K 32 KB + V 2 x 32 KB + P 32 KB of shared
// memory, 256 TMEM columns (S, O).
#include <algorithm>

#include "tbik_common.cuh"
#include "tbik_internal.h"

namespace tbik_b200 {

// tbik_gemm_tc.cu: bf16 3-D tensor map, 128-byte swizzle
tbik_status tc_make_map_3d_bf16_sw128(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1);

namespace {

constexpr int T5_Q = 128;               // queries per CTA
constexpr int T5_K = 128;               // keys per block
constexpr int T5_D = 128;               // head dim
constexpr int T5_ATOM = 128 * 128;      // one [128 rows][64 bf16] SW128 box: 16 KB
constexpr int T5_TILE = 2 * T5_ATOM;    // a [128][128] bf16 operand: 32 KB
constexpr int T5_SMEM = 5 * T5_TILE + 1024 + 256;

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ uint64_t t5_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

__global__ void __launch_bounds__(128, 1)
    attn_tc5_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, int S, int nq, int nkv, float scale_log2,
                    uint16_t* __restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t t5_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(t5_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sK = sm + T5_TILE;
  uint8_t* sV = sm + 2 * T5_TILE;  // two buffers
  uint8_t* sP = sm + 4 * T5_TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + 5 * T5_TILE);  // [2]: K_j + V_j (+ Q) landed
  uint64_t* sbar = full + 2;                                       // S MMA of the block done
  uint64_t* obar = sbar + 1;                                       // O MMA of the block done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(obar + 1);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int qb = static_cast<int>(gridDim.z) - 1 - static_cast<int>(blockIdx.z);  // heaviest blocks first
  const int h = blockIdx.x, b = blockIdx.y;
  const int kh = h / (nq / nkv);
  const int row = qb * T5_Q + tid;  // this thread's query
  const int nkb = qb + 1;           // causal key blocks

  if (tid == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(sbar, 1);
    mbar_init(obar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tS = tbase, tO = tbase + 128;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  pdl_wait();
  pdl_trigger();

  auto load_kv = [&](int j, int vb, bool with_q) {
    mbar_arrive_expect_tx(&full[vb], static_cast<uint32_t>((with_q ? 3 : 2) * T5_TILE));
    if (with_q)
      for (int a = 0; a < 2; ++a) tma_load_3d(sQ + a * T5_ATOM, &tmQ, &full[vb], h * T5_D + a * 64, qb * T5_Q, b);
    for (int a = 0; a < 2; ++a) {
      tma_load_3d(sK + a * T5_ATOM, &tmK, &full[vb], kh * T5_D + a * 64, j * T5_K, b);
      tma_load_3d(sV + vb * T5_TILE + a * T5_ATOM, &tmV, &full[vb], kh * T5_D + a * 64, j * T5_K, b);
    }
  };
  if (tid == 0) load_kv(0, 0, true);

  constexpr uint32_t IDESC_S = umma_idesc_bf16(128, 128, 0, 0);
  constexpr uint32_t IDESC_O = umma_idesc_bf16(128, 128, 0, 1);
  const float NEG_INF = __int_as_float(0xFF800000);
  float m = NEG_INF, l = 0.0f;

  for (int j = 0; j < nkb; ++j) {
    const int vb = j & 1;
    // ---- S = Q . K_j^T -------------------------------------------------------------
    if (tid == 0) {
      mbar_wait(&full[vb], (j >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < T5_D / 16; ++kk) {  // K-major A and B: +32 B per step, atom every 4
        const uint32_t off = (kk >> 2) * T5_ATOM + (kk & 3) * 32;
        umma_bf16(tS, t5_desc(smem_u32(sQ) + off, 16, 1024), t5_desc(smem_u32(sK) + off, 16, 1024), IDESC_S,
                  kk != 0 ? 1u : 0u);
      }
      umma_commit(sbar);
    }
    __syncwarp();
    mbar_wait(sbar, j & 1);
    tc_fence_after();
    // ---- row softmax (thread = query row = TMEM lane) --------------------------------
    float s[T5_K];
#pragma unroll
    for (int c = 0; c < T5_K / 32; ++c) {
      float t[32];
      tmem_ld32(tS + lane_off + c * 32, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) s[c * 32 + i] = t[i];
    }
    float bm = NEG_INF;
#pragma unroll
    for (int i = 0; i < T5_K; ++i) {
      const int key = j * T5_K + i;
      if (key > row || key >= S) s[i] = NEG_INF;
      bm = fmaxf(bm, s[i]);
    }
    const float mn = fmaxf(m, bm);
    const float mc = mn == NEG_INF ? 0.0f : __fmul_rn(mn, scale_log2);
    const float alpha = m == NEG_INF ? 0.0f : exp2f(__fsub_rn(__fmul_rn(m, scale_log2), mc));
    m = mn;
    float ps = 0.0f;
    uint32_t pk[T5_K / 2];
#pragma unroll
    for (int i = 0; i < T5_K; i += 2) {
      const float p0 = exp2f(__fsub_rn(__fmul_rn(s[i], scale_log2), mc));
      const float p1 = exp2f(__fsub_rn(__fmul_rn(s[i + 1], scale_log2), mc));
      ps = __fadd_rn(__fadd_rn(ps, p0), p1);
      pk[i / 2] = static_cast<uint32_t>(f32_to_bf16_bits(p0)) | (static_cast<uint32_t>(f32_to_bf16_bits(p1)) << 16);
    }
    l = __fadd_rn(__fmul_rn(l, alpha), ps);
    // ---- the previous O MMA is done: P / V buffers free, O stable --------------------
    if (j > 0) {
      mbar_wait(obar, (j - 1) & 1);
      tc_fence_after();
      // (warp-uniform: the TMEM loads / stores are warp-collective; alpha = 1 rows
      // are multiplied by 1, exactly)
      if (__any_sync(0xffffffffu, alpha != 1.0f)) {
#pragma unroll
        for (int c = 0; c < T5_D / 32; ++c) {
          float o[32];
          tmem_ld32(tO + lane_off + c * 32, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __fmul_rn(o[i], alpha);
          tmem_st32(tO + lane_off + c * 32, o);
        }
        tmem_wait_st();
      }
    }
    // next block's K (the S MMA read it) and V (other buffer, its O MMA is done)
    if (tid == 0 && j + 1 < nkb) load_kv(j + 1, vb ^ 1, false);
    // P row -> shared memory, K-major SW128 ([128 rows][64 keys] atoms, 16-byte chunk
    // c of row r at chunk c ^ (r & 7))
#pragma unroll
    for (int c = 0; c < T5_K / 8; ++c) {
      uint8_t* dst = sP + (c >> 3) * T5_ATOM + tid * 128 + (((c & 7) ^ (tid & 7)) * 16);
      *reinterpret_cast<uint4*>(dst) = make_uint4(pk[c * 4], pk[c * 4 + 1], pk[c * 4 + 2], pk[c * 4 + 3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    // ---- O += P . V_j -----------------------------------------------------------------
    if (tid == 0) {
      tc_fence_after();
      const uint32_t vbase = smem_u32(sV + vb * T5_TILE);
#pragma unroll
      for (int kk = 0; kk < T5_K / 16; ++kk) {
        // A = P K-major (+32 B per step, atom every 4); B = V MN-major: 64-dim atoms 16 KB
        // apart (LBO), 8-key groups 1 KB apart (SBO), +16 keys (2 KB) per step
        const uint32_t aoff = (kk >> 2) * T5_ATOM + (kk & 3) * 32;
        umma_bf16(tO, t5_desc(smem_u32(sP) + aoff, 16, 1024), t5_desc(vbase + kk * 2048, T5_ATOM, 1024), IDESC_O,
                  (j | kk) != 0 ? 1u : 0u);
      }
      umma_commit(obar);
    }
    __syncwarp();
  }
  mbar_wait(obar, (nkb - 1) & 1);
  tc_fence_after();
  {
    uint16_t* op = out + (static_cast<int64_t>(b) * S + min(row, S - 1)) * ldo + h * T5_D;
#pragma unroll
    for (int c = 0; c < T5_D / 32; ++c) {
      float o[32];
      tmem_ld32(tO + lane_off + c * 32, o);  // all lanes (warp-collective); rows >= S store nothing
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          w[e] = static_cast<uint32_t>(f32_to_bf16_bits(__fdiv_rn(o[i + 2 * e], l))) |
                 (static_cast<uint32_t>(f32_to_bf16_bits(__fdiv_rn(o[i + 2 * e + 1], l))) << 16);
        if (row < S) *reinterpret_cast<uint4*>(op + c * 32 + i) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 256);
  }
}

}  // namespace

// q [batch*S][ldq], k / v [batch*S][ldk / ldv] bf16, head_dim 128 (checked by the caller).
tbik_status launch_attn_tc5(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                            int64_t batch, int S, int nq, int nkv, float scale_log2, void* out, int64_t ldo,
                            cudaStream_t s) {
  CUtensorMap mQ, mK, mV;
  const uint64_t Sb = static_cast<uint64_t>(S);
  TBIK_TRY(tc_make_map_3d_bf16_sw128(&mQ, q, static_cast<uint64_t>(nq) * T5_D, Sb, static_cast<uint64_t>(batch),
                                     static_cast<uint64_t>(ldq) * 2, static_cast<uint64_t>(ldq) * 2 * Sb, 64, T5_Q));
  TBIK_TRY(tc_make_map_3d_bf16_sw128(&mK, k, static_cast<uint64_t>(nkv) * T5_D, Sb, static_cast<uint64_t>(batch),
                                     static_cast<uint64_t>(ldk) * 2, static_cast<uint64_t>(ldk) * 2 * Sb, 64, T5_K));
  TBIK_TRY(tc_make_map_3d_bf16_sw128(&mV, v, static_cast<uint64_t>(nkv) * T5_D, Sb, static_cast<uint64_t>(batch),
                                     static_cast<uint64_t>(ldv) * 2, static_cast<uint64_t>(ldv) * 2 * Sb, 64, T5_K));
  TBIK_CUDA(cudaFuncSetAttribute(attn_tc5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, T5_SMEM));
  dim3 grid(static_cast<unsigned>(nq), static_cast<unsigned>(batch), static_cast<unsigned>((S + T5_Q - 1) / T5_Q));
  TBIK_CUDA(launch_pdl(attn_tc5_kernel, grid, dim3(128), static_cast<size_t>(T5_SMEM), s, mQ, mK, mV, S, nq, nkv,
                       scale_log2, static_cast<uint16_t*>(out), ldo));
  count_launch("attn_tc5_kernel");
  return TBIK_OK;
}

}  // namespace tbik_b200
