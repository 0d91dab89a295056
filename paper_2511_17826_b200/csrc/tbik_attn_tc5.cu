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
constexpr int T5_THREADS = 512;         // 16 warps: 4 column quarters x 4 TMEM lane groups
// Q, K x 2, V x 2, P tiles; row max / sum partials [4 quarters][128 rows] x 2; barriers
constexpr int T5_SMEM = 6 * T5_TILE + 1024 + 2 * 4 * 128 * 4 + 128;

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

// The four warps that share TMEM lane group g (warps g, g + 4, g + 8, g + 12: the four
// column quarters of the same 32 query rows) meet on named barrier 1 + g.
__device__ __forceinline__ void row_group_sync(int g) {
  asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
}

__global__ void __launch_bounds__(T5_THREADS, 1)
    attn_tc5_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, int S, int nq, int nkv, float scale_log2,
                    uint16_t* __restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t t5_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(t5_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sK = sm + T5_TILE;      // two buffers
  uint8_t* sV = sm + 3 * T5_TILE;  // two buffers
  uint8_t* sP = sm + 5 * T5_TILE;
  float* red_max = reinterpret_cast<float*>(sm + 6 * T5_TILE);  // [quarter][row]
  float* red_sum = red_max + 4 * 128;
  uint64_t* kfull = reinterpret_cast<uint64_t*>(red_sum + 4 * 128);  // [2]: K_j (+ Q) landed
  uint64_t* vfull = kfull + 2;                                       // [2]: V_j landed
  uint64_t* sbar = vfull + 2;                                        // [2]: S MMA of block j done
  uint64_t* obar = sbar + 2;                                         // O MMA of the block done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(obar + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = warp & 3;   // TMEM lane group (warp % 4 may access lanes 32 grp .. 32 grp + 31)
  const int qtr = warp >> 2;  // column quarter of S / O this thread handles
  const int r = grp * 32 + lane;
  const int qb = static_cast<int>(gridDim.z) - 1 - static_cast<int>(blockIdx.z);  // heaviest blocks first
  const int h = blockIdx.x, b = blockIdx.y;
  const int kh = h / (nq / nkv);
  const int row = qb * T5_Q + r;  // this thread's query
  const int nkb = qb + 1;         // causal key blocks

  if (tid == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < 7; ++i) mbar_init(&kfull[i], 1);  // kfull, vfull, sbar, obar
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tO = tbase + 256;  // S_j at tbase + 128 (j & 1)
  const uint32_t lane_off = static_cast<uint32_t>(grp * 32) << 16;
  pdl_wait();
  pdl_trigger();

  auto load_k = [&](int j, bool with_q) {
    uint64_t* bar = &kfull[j & 1];
    mbar_arrive_expect_tx(bar, static_cast<uint32_t>((with_q ? 2 : 1) * T5_TILE));
    if (with_q)
      for (int a = 0; a < 2; ++a) tma_load_3d(sQ + a * T5_ATOM, &tmQ, bar, h * T5_D + a * 64, qb * T5_Q, b);
    for (int a = 0; a < 2; ++a)
      tma_load_3d(sK + (j & 1) * T5_TILE + a * T5_ATOM, &tmK, bar, kh * T5_D + a * 64, j * T5_K, b);
  };
  auto load_v = [&](int j) {
    uint64_t* bar = &vfull[j & 1];
    mbar_arrive_expect_tx(bar, static_cast<uint32_t>(T5_TILE));
    for (int a = 0; a < 2; ++a)
      tma_load_3d(sV + (j & 1) * T5_TILE + a * T5_ATOM, &tmV, bar, kh * T5_D + a * 64, j * T5_K, b);
  };
  constexpr uint32_t IDESC_S = umma_idesc_bf16(128, 128, 0, 0);
  constexpr uint32_t IDESC_O = umma_idesc_bf16(128, 128, 0, 1);
  auto issue_s = [&](int j) {  // S_j = Q . K_j^T into TMEM buffer j & 1 (one thread)
    mbar_wait(&kfull[j & 1], (j >> 1) & 1);
    tc_fence_after();
    const uint32_t kbase = smem_u32(sK + (j & 1) * T5_TILE);
#pragma unroll
    for (int kk = 0; kk < T5_D / 16; ++kk) {  // K-major A and B: +32 B per step, atom every 4
      const uint32_t off = (kk >> 2) * T5_ATOM + (kk & 3) * 32;
      umma_bf16(tbase + (j & 1) * 128, t5_desc(smem_u32(sQ) + off, 16, 1024), t5_desc(kbase + off, 16, 1024),
                IDESC_S, kk != 0 ? 1u : 0u);
    }
    umma_commit(&sbar[j & 1]);
  };
  if (tid == 0) {
    load_k(0, true);
    load_v(0);
    if (nkb > 1) {
      load_k(1, false);
      load_v(1);
    }
    issue_s(0);
  }

  const float NEG_INF = __int_as_float(0xFF800000);
  float m = NEG_INF, l = 0.0f;

  for (int j = 0; j < nkb; ++j) {
    // ---- S_{j+1} into the other TMEM buffer (its S_{j-1} was read before the last
    // block's closing barrier), overlapping this block's softmax --------------------
    if (tid == 0 && j + 1 < nkb) issue_s(j + 1);
    __syncwarp();
    mbar_wait(&sbar[j & 1], (j >> 1) & 1);
    tc_fence_after();
    // K buffer j & 1 is free once S_j is done
    if (tid == 0 && j + 2 < nkb) load_k(j + 2, false);
    // ---- row softmax: 4 threads per query row (TMEM lane), 32 keys each -------------
    float s[32];
    tmem_ld32(tbase + (j & 1) * 128 + lane_off + qtr * 32, s);
    // only the diagonal block holds keys past the query (or past the sequence end:
    // qb * 128 < S, so every earlier block lies inside it)
    if (j == qb) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int key = j * T5_K + qtr * 32 + i;
        if (key > row || key >= S) s[i] = NEG_INF;
      }
    }
    float bm = NEG_INF;
#pragma unroll
    for (int i = 0; i < 32; ++i) bm = fmaxf(bm, s[i]);
    red_max[qtr * 128 + r] = bm;
    row_group_sync(grp);
    bm = fmaxf(fmaxf(red_max[r], red_max[128 + r]), fmaxf(red_max[256 + r], red_max[384 + r]));
    const float mn = fmaxf(m, bm);
    const float mc = mn == NEG_INF ? 0.0f : __fmul_rn(mn, scale_log2);
    const float alpha = m == NEG_INF ? 0.0f : exp2f(__fsub_rn(__fmul_rn(m, scale_log2), mc));
    m = mn;
    float ps = 0.0f;  // this quarter's keys in order
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float p0 = exp2f(__fsub_rn(__fmul_rn(s[i], scale_log2), mc));
      const float p1 = exp2f(__fsub_rn(__fmul_rn(s[i + 1], scale_log2), mc));
      ps = __fadd_rn(__fadd_rn(ps, p0), p1);
      pk[i / 2] = bf16x2_bits(p0, p1);
    }
    red_sum[qtr * 128 + r] = ps;
    row_group_sync(grp);
    // block sum: the four quarter sums in quarter order (the same in all four threads)
    ps = __fadd_rn(__fadd_rn(__fadd_rn(red_sum[r], red_sum[128 + r]), red_sum[256 + r]), red_sum[384 + r]);
    l = __fadd_rn(__fmul_rn(l, alpha), ps);
    // ---- the previous O MMA is done: P and V buffer (j+1)&1 free, O stable ------------
    if (j > 0) {
      mbar_wait(obar, (j - 1) & 1);
      tc_fence_after();
      if (tid == 0 && j + 1 < nkb) load_v(j + 1);
      // (warp-uniform: the TMEM loads / stores are warp-collective; alpha = 1 rows
      // are multiplied by 1, exactly)
      if (__any_sync(0xffffffffu, alpha != 1.0f)) {
        float o[32];
        tmem_ld32(tO + lane_off + qtr * 32, o);
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = __fmul_rn(o[i], alpha);
        tmem_st32(tO + lane_off + qtr * 32, o);
        tmem_wait_st();
      }
    }
    // this quarter of the P row -> shared memory, K-major SW128 ([128 rows][64 keys]
    // atoms, 16-byte chunk c of row r at chunk c ^ (r & 7))
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int c = qtr * 4 + cc;
      uint8_t* dst = sP + (c >> 3) * T5_ATOM + r * 128 + (((c & 7) ^ (r & 7)) * 16);
      *reinterpret_cast<uint4*>(dst) = make_uint4(pk[cc * 4], pk[cc * 4 + 1], pk[cc * 4 + 2], pk[cc * 4 + 3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    // ---- O += P . V_j -----------------------------------------------------------------
    if (tid == 0) {
      mbar_wait(&vfull[j & 1], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t vbase = smem_u32(sV + (j & 1) * T5_TILE);
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
    uint16_t* op = out + (static_cast<int64_t>(b) * S + min(row, S - 1)) * ldo + h * T5_D + qtr * 32;
    float o[32];
    tmem_ld32(tO + lane_off + qtr * 32, o);  // all lanes (warp-collective); rows >= S store nothing
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w[e] = bf16x2_bits(__fdiv_rn(o[i + 2 * e], l), __fdiv_rn(o[i + 2 * e + 1], l));
      if (row < S) *reinterpret_cast<uint4*>(op + i) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
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
  TBIK_CUDA(launch_pdl(attn_tc5_kernel, grid, dim3(T5_THREADS), static_cast<size_t>(T5_SMEM), s, mQ, mK, mV, S, nq, nkv,
                       scale_log2, static_cast<uint16_t*>(out), ldo));
  count_launch("attn_tc5_kernel");
  return TBIK_OK;
}

}  // namespace tbik_b200
