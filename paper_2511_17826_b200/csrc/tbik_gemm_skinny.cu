// tbik_gemm_skinny.cu -- the tensor-core-leaf TBIK GEMM for skinny activations
// (decode-sized M <= 128), where the weight stream is the whole cost.
//
// Swap-AB: the MMA's 128-row operand is a 128-column slice of the WEIGHTS
// (W[K x N] row-major = MN-major A, read by TMA exactly as the wide kernel reads
// B) and the tokens are the MMA N dimension (MT = 16/32/64/128, K-major B = X rows).
// D[n][m] = sum_k W[k][n] X[m][k] lands in TMEM with lane = weight column and
// column = token, so a leaf drains MT x 4 bytes per lane instead of the
// 128-row padded tile of the wide kernel (tbik_gemm_tc.cu), and shared memory
// goes to weight stages.
//
// The per-element arithmetic is the wide kernel's: the leaf P_t is block_k/16
// tcgen05 kind::f16 MMAs (K = 16 each) into a zeroed f32 accumulator -- each
// output element is the same 16-product K steps in the same order; only which
// operand sits in the A slot differs, and the product a*b is commutative
// (checked bit for bit against the wide kernel over every shape class in
// tests/test_gpu_gemm.py::test_skinny_*).  Above the leaf everything is the
// reference's reduction in its order:
//   level 0   g = ((0 + P_0) + P_1) + ... + P_{kf-1}         (matmul.cpp:100-125)
//   levels>=1 binary counter over group values, new + old     (matmul.cpp:107-123)
//   units     when the tiles alone leave SMs idle, the K range of a tile is cut
//             into X <= 8 aligned 2^j-group subtrees (or, for a view of few
//             groups -- a TP shard --, its single leaves), one per CTA of a
//             thread-block cluster of X CTAs.  Each CTA leaves its unit value in
//             shared memory; after a cluster barrier CTA u evaluates rows
//             [u R, u R + R) of the tile over all X values read through DSMEM, in
//             the fold + contiguous-halves tree order (oracle.cpp:11-20,
//             Theorem 1).  No workspace, no second launch.
//   pairs     (p.pair) a tile whose K range is ONE leaf group runs on a CTA
//             pair: the leading CTA folds the first leaves, sends the prefix by
//             st.async into the partner's shared memory (completing on its
//             mbarrier), the partner continues the fold over its last <= NACC
//             leaves kept in TMEM -- the same sequential level-0 order split at a
//             leaf; two subtree units hand over the same way, (0 + v1) + (0 + v0).
//
// Warp roles (one CTA per SM; persistent over tiles when X = 1):
//   warp 0  TMA producer: per stage {W KS k x BNW n (64-column SW128 atoms, or one
//           32-column SW64 atom), X MT x KS k as KS / 64 boxes}
//   warp 1  MMA issuer (one elected thread), NACC TMEM accumulators in rotation
//   warp 2  TMEM allocator (512 columns: accumulators + tree levels 1..levels)
//   warps 4.. merge warps: thread (q, lane) owns weight column n0 + q LPQ + lane
//             for TPW <= 32 tokens (TMEM lane quarter q); MT / 8 warps.
// Launched with programmatic dependent launch (griddepcontrol.wait before the
// first operand / output access, dependents triggered after the last load).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <cstdio>
#include <string>
#include <vector>

#include "tbik_common.cuh"
#include "tbik_internal.h"

namespace tbik_b200 {

// tbik_gemm_tc.cu (tensor-map helpers shared by the tcgen05 kernels)
tbik_status tc_make_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
tbik_status tc_make_map_2d_sw64(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                                uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);

namespace {

constexpr int SK_BN = 128;                  // weight columns per tile (BNW = 128: MMA M = 128)
constexpr int SK_KSTAGE = 64;               // K granularity of a stage (KS = 64 or 128 per stage)
constexpr int SK_TMEM_COLS = 512;
constexpr int SK_SMEM_LIMIT = 232448;
constexpr int SK_MAX_UNITS = 8;
constexpr int SK_MAX_M = 128;    // tokens = MMA N (16 / 32 / 64 / 128)  // K-split units = CTAs of one cluster (portable cluster size)

// Tokens per merge thread (TPW) and merge warps (4 lane quarters x MT / TPW):
// <= 32 tokens per thread, so the per-tile tail (fold, stores) is spread over
// MT / 8 warps (TPW = 64 measured slower at M = 64 / 128).
template <int MT>
constexpr int sk_tpw() { return MT > 32 ? 32 : MT; }
template <int MT>
constexpr int sk_merge_warps() { return 4 * (MT / sk_tpw<MT>()); }
template <int MT>
constexpr int sk_threads() { return 128 + 32 * sk_merge_warps<MT>(); }
template <int MT>
constexpr int sk_nacc() { return MT >= 128 ? 2 : 4; }
// BNW = weight columns per tile: 128 (MMA M = 128, all TMEM lanes) or 64 (MMA
// M = 64: rows land in TMEM lanes 0-15 of each 32-lane quarter, CUTLASS
// mma_traits_sm100.hpp "half subpartitions" atom) -- twice the tiles for short K.
// KS = K rows per stage: the W box is {64 columns, KS rows} (one SW128 atom column
// of KS / 8 1-KB row groups); X arrives as KS / 64 boxes of {64 K, MT tokens}.
// Taller W boxes stream faster from L2 (tools/micro/tma_ingest.cu: the time of an
// L2-resident shard follows the number of boxes, not their bytes).
template <int KS>
constexpr int sk_w_atom() { return 64 * KS * 2; }
template <int BNW, int KS = 64>
constexpr int sk_w_stage() { return BNW * KS * 2; }
template <int MT, int KS = 64>
constexpr int sk_x_stage() { return MT * 128 * (KS / 64); }
// Pair mode (MT <= 64): the finishing CTA receives its partner's prefix fold,
// [BNW columns][MT tokens] f32.  (At MT = 128 -- two accumulators, so a 5 + 2
// leaf split, 4 stages -- it measured slower: TP = 8 shard 11.2 vs 9.9 us.)
template <int MT, int BNW>
constexpr bool sk_pair_ok() { return MT <= 64; }
template <int MT, int BNW>
constexpr int sk_prefix_bytes() { return sk_pair_ok<MT, BNW>() ? BNW * MT * 4 : 0; }
template <int MT, int BNW = 128, int KS = 64>
constexpr int sk_stages() {
  return (SK_SMEM_LIMIT - 2048 - sk_prefix_bytes<MT, BNW>()) / (sk_w_stage<BNW, KS>() + sk_x_stage<MT, KS>());
}
template <int MT, int BNW = 128, int KS = 64>
constexpr size_t sk_smem() {
  return 1024 + static_cast<size_t>(sk_stages<MT, BNW, KS>()) * (sk_w_stage<BNW, KS>() + sk_x_stage<MT, KS>()) +
         sk_prefix_bytes<MT, BNW>() + 512;
}
static_assert(sk_smem<16>() <= SK_SMEM_LIMIT && sk_smem<32>() <= SK_SMEM_LIMIT && sk_smem<64>() <= SK_SMEM_LIMIT &&
                  sk_smem<128>() <= SK_SMEM_LIMIT && sk_smem<16, 64>() <= SK_SMEM_LIMIT &&
                  sk_smem<128, 64>() <= SK_SMEM_LIMIT && sk_smem<128, 128, 128>() <= SK_SMEM_LIMIT &&
                  sk_stages<128, 128, 128>() >= 3,
              "skinny smem budget");
// Tree levels that fit in TMEM next to the accumulators.
template <int MT>
constexpr int sk_max_levels() { return SK_TMEM_COLS / MT - sk_nacc<MT>(); }

struct SkParams {
  int M, N, K;
  int bk, kf, T;
  int ntiles;
  int units;           // X: values per tile handed to the finish (1 = the item's value is final)
  int pair;            // CTA-pair handoff instead of the cluster finish (units = 2, see the kernel):
                       // 1 = one leaf group split at a leaf, 2 = two subtree units
  int tiles_per_unit;  // leaves per unit
  int levels;          // tree levels inside a unit (log2 of its groups; 0 for leaf units)
  int fold;            // finish: level-0 fold length over unit values (kf for leaf units, else 1)
  int log_groups;      // finish: log2(units / fold)
  long long items;
  int bn;              // weight columns per tile (the kernel's BNW)
  float* out;
  long long ldo;
  unsigned long long* trace;  // diagnostics (knob sk_trace): per-CTA phase clocks, else null
};

__device__ __forceinline__ void tmem_ld16r(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld16_dep(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
// Whole-cluster barrier (a lone CTA is a cluster of one).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_map(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 dsmem_ld_f32x4(uint32_t addr) {
  float4 v;
  // not volatile: the data is published by the cluster barrier (which carries the
  // memory clobber), so the loads of several items may be scheduled together
  asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(addr));
  return v;
}

struct SkItem {
  int n0, unit, t_begin, t_end;
};
// Units of one tile are adjacent items, so they run in the same wave and the
// tile's finish starts as soon as its slowest unit is done.
__device__ __forceinline__ SkItem sk_decode(const SkParams& p, long long item) {
  SkItem it;  // 32-bit division (items < 2^31, checked at launch)
  const uint32_t i = static_cast<uint32_t>(item), u = static_cast<uint32_t>(p.units);
  it.unit = static_cast<int>(i % u);
  it.n0 = static_cast<int>(i / u) * p.bn;
  it.t_begin = it.unit * p.tiles_per_unit;
  it.t_end = min(p.T, it.t_begin + p.tiles_per_unit);
  return it;
}
template <int KS>
__device__ __forceinline__ int sk_chunks(const SkParams& p, int t) {
  const int kt0 = t * p.bk;
  const int kh = (kt0 + p.bk <= p.K) ? p.bk : p.K - kt0;
  return (kh + KS - 1) / KS;
}

// In-cluster finish of a K-split tile (see the kernel).  UNITS > 0: a compile-time
// unit count, so the once-per-CTA code holds only what this split runs (its
// instructions are fetched cold); UNITS = 0: any count <= SK_MAX_UNITS.
template <int UNITS, int BNW>
__device__ __forceinline__ void sk_finish(const SkParams& p, const uint8_t* sW) {
  constexpr int UMAX = UNITS > 0 ? UNITS : SK_MAX_UNITS;
  const int nu = UNITS > 0 ? UNITS : p.units;
  // work items: (row, 4-column quad) of this CTA's row slice, 16-byte DSMEM loads
  // from every unit, spread over all warps (their roles are done), two items in
  // flight per thread
  const int tid = threadIdx.x;
  const int unit = static_cast<int>(blockIdx.x % nu);
  const int n0 = static_cast<int>(blockIdx.x / nu) * BNW;
  const int R = (p.M + nu - 1) / nu;
  const int m_lo = unit * R, m_hi = min(p.M, m_lo + R);
  const int nitems = (m_hi > m_lo ? m_hi - m_lo : 0) * (BNW / 4);
  const uint32_t fb = smem_u32(sW);
  uint32_t peer[UMAX];
#pragma unroll
  for (int x = 0; x < UMAX; ++x) peer[x] = x < nu ? dsmem_map(fb, static_cast<uint32_t>(x)) : 0u;
#pragma unroll 2
  for (int idx = tid; idx < nitems; idx += static_cast<int>(blockDim.x)) {
    const int m = m_lo + idx / (BNW / 4);
    const int c4 = (idx % (BNW / 4)) * 4;
    const uint32_t off = static_cast<uint32_t>((m * BNW + c4) * 4);
    float4 vals[UMAX];
#pragma unroll
    for (int x = 0; x < UMAX; ++x)
      vals[x] = x < nu ? dsmem_ld_f32x4(peer[x] + off) : make_float4(0.f, 0.f, 0.f, 0.f);
    float res[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // level-0 fold over `fold` consecutive values, then the contiguous-halves
      // tree over the groups (binary counter, new + old)
      float stack[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      float acc = 0.0f;
      int gcount = 0, in_fold = 0;
#pragma unroll
      for (int x = 0; x < UMAX; ++x) {
        if (x < nu) {
          const float vx = j == 0 ? vals[x].x : j == 1 ? vals[x].y : j == 2 ? vals[x].z : vals[x].w;
          acc = __fadd_rn(acc, vx);
          if (++in_fold == p.fold) {
            float v = acc;
            int l = 0;
#pragma unroll
            for (int b = 0; b < 3; ++b)
              if (((gcount >> b) & 1) && l == b) {
                v = __fadd_rn(v, stack[b]);
                l = b + 1;
              }
#pragma unroll
            for (int b = 0; b < 4; ++b)
              if (l == b) stack[b] = v;
            ++gcount;
            in_fold = 0;
            acc = 0.0f;
          }
        }
      }
      res[j] = stack[0];
#pragma unroll
      for (int b = 1; b < 4; ++b)
        if (b == p.log_groups) res[j] = stack[b];
    }
    const int n = n0 + c4;
    float* dst = p.out + static_cast<size_t>(m) * p.ldo + n;
    if (n + 3 < p.N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      *reinterpret_cast<float4*>(dst) = make_float4(res[0], res[1], res[2], res[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (n + j < p.N) dst[j] = res[j];
    }
  }
}

template <int MT, int BNW, int KS>
__global__ void __launch_bounds__(sk_threads<MT>(), 1)
    tc_skinny_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                     const SkParams p) {
  constexpr int NST = sk_stages<MT, BNW, KS>();
  constexpr int W_ATOM = sk_w_atom<KS>();
  constexpr int W_STAGE = sk_w_stage<BNW, KS>();
  // MMA M = 64 for BNW = 32 (the rows past the tile are a repeat of its 32-column
  // atom, computed and never read); TMEM lanes holding rows per 32-lane quarter:
  constexpr int MMA_M = BNW < 64 ? 64 : BNW;
  constexpr int LPQ = MMA_M / 4;
  constexpr int NACC = sk_nacc<MT>();
  constexpr int X_BOX = MT * 128;
  constexpr int X_STAGE = sk_x_stage<MT, KS>();
  constexpr uint32_t TX_BYTES = W_STAGE + X_STAGE;
  constexpr uint32_t IDESC = umma_idesc_bf16(MMA_M, MT, /*a_mn_major=*/1, /*b_mn_major=*/0);
  constexpr int TPW = sk_tpw<MT>();
  constexpr int NMW = sk_merge_warps<MT>();
  constexpr int NCH = TPW / 16;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = sW + NST * W_STAGE;
  float* sPre = reinterpret_cast<float*>(sX + NST * X_STAGE);  // pair mode: partner's prefix
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + NST * X_STAGE + sk_prefix_bytes<MT, BNW>());
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + NACC;
  uint64_t* pre_full = tempty + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pre_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long t0 = clock64();
#define SK_TRACE(i) \
  if (p.trace) p.trace[blockIdx.x * 16 + (i)] = static_cast<unsigned long long>(clock64() - t0)

  if (warp == 0 && lane == 0) {
    if (p.trace) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      p.trace[blockIdx.x * 16 + 15] = gt;
    }
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], NMW);  // every merge warp
    }
    mbar_init(pre_full, 1);
    fence_barrier_init();
    // pair mode, finishing CTA: the partner's prefix arrives by st.async
    if (p.pair && (blockIdx.x & 1)) mbar_arrive_expect_tx(pre_full, static_cast<uint32_t>(sk_prefix_bytes<MT, BNW>()));
  }
  if (warp == 2) tmem_alloc(tmem_slot, SK_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // pair mode: the partner's barrier must be initialised before the leading CTA
  // writes to it -- arrive now (relaxed: nothing to publish but the barrier
  // init, fenced above), wait only right before the remote stores.
  if (p.pair) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  // Programmatic dependent launch: the prologue above (barriers, TMEM, descriptor
  // prefetch, instruction fetch) may overlap the previous kernel's tail; operands
  // and the output are touched only after that kernel has completed (a no-op when
  // launched without the attribute).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) SK_TRACE(1);

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (long long item = blockIdx.x; item < p.items; item += gridDim.x) {
        const SkItem it = sk_decode(p, item);
        for (int t = it.t_begin; t < it.t_end; ++t) {
          const int nch = sk_chunks<KS>(p, t);
          for (int c = 0; c < nch; ++c) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], TX_BYTES);
            const int k = t * p.bk + c * KS;
            uint8_t* w = sW + stage * W_STAGE;
            tma_load_2d(w, &tmW, &full[stage], it.n0, k);
            if constexpr (BNW == 128) tma_load_2d(w + W_ATOM, &tmW, &full[stage], it.n0 + 64, k);
#pragma unroll
            for (int j = 0; j < KS / 64; ++j)
              tma_load_2d(sX + stage * X_STAGE + j * X_BOX, &tmX, &full[stage], k + 64 * j, 0);
            if (p.trace && c == 0 && t == it.t_begin && item == blockIdx.x) SK_TRACE(2);
            if (++stage == NST) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      SK_TRACE(3);
      // Every load of this CTA is issued: the next kernel may begin its prologue
      // (dependents launch once every CTA of this grid has triggered or exited, so
      // later-wave CTAs are never starved of SMs).
      asm volatile("griddepcontrol.launch_dependents;");
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc_iter = 0;
      for (long long item = blockIdx.x; item < p.items; item += gridDim.x) {
        const SkItem it = sk_decode(p, item);
        for (int t = it.t_begin; t < it.t_end; ++t, ++acc_iter) {
          const int buf = acc_iter % NACC;
          const uint32_t use = acc_iter / NACC;
          mbar_wait(&tempty[buf], (use & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + buf * MT;
          const int nch = sk_chunks<KS>(p, t);
          for (int c = 0; c < nch; ++c) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (p.trace && c == 0 && t == it.t_begin && item == blockIdx.x) SK_TRACE(4);
            const uint32_t w_base = smem_u32(sW + stage * W_STAGE);
            const uint32_t x_base = smem_u32(sX + stage * X_STAGE);
#pragma unroll
            for (int kk = 0; kk < KS / 16; ++kk) {
              // A = W: MN-major SW128, two 64-column atoms W_ATOM apart (LBO), 8-row K
              // groups 1 KB apart (SBO), +16 K rows (2 KB) per step.
              uint64_t adesc;
              if constexpr (BNW == 32)  // SW64 MN-major: one 32-column atom (LBO 0), +1 KB per step
                adesc = (umma_desc_sw128(w_base + kk * 1024, 0, 512) & ~(uint64_t{7} << 61)) | (uint64_t{4} << 61);
              else
                adesc = umma_desc_sw128(w_base + kk * 2048, W_ATOM, 1024);
              // B = X: K-major SW128, one box per 64 K, +32 B per 16-element K step
              // inside the 128 B row.
              const uint64_t bdesc = umma_desc_sw128(x_base + (kk >> 2) * X_BOX + (kk & 3) * 32, 16, 1024);
              umma_bf16(d, adesc, bdesc, IDESC, (c | kk) != 0 ? 1u : 0u);
            }
            umma_commit(&empty[stage]);
            if (++stage == NST) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(&tfull[buf]);
        }
      }
      SK_TRACE(5);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = (warp - 4) & 3;         // TMEM lane quarter
    const int h0 = ((warp - 4) >> 2) * TPW;  // first token of this warp
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + h0;
    float g[TPW];
    uint32_t acc_iter = 0;
    for (long long item = blockIdx.x; item < p.items; item += gridDim.x) {
      const SkItem it = sk_decode(p, item);
      const int n = it.n0 + q * LPQ + lane;
      // BNW = 64: lanes 16-31 of a quarter hold no row; BNW = 32: nor quarters 2-3
      const bool lane_ok = lane < LPQ && q * LPQ < BNW;
      if constexpr (sk_pair_ok<MT, BNW>()) {
        if (p.pair == 1 && it.unit == 1) {
          // Pair mode 1, finishing CTA: its leaves (<= NACC, one accumulator each,
          // kept in TMEM) continue the partner's prefix fold in leaf order:
          // ((prefix + l_a) + l_a+1) + ... -- the sequential level-0 fold of the
          // group (matmul.cpp:101-103), split at a leaf boundary.
          const int nl = it.t_end - it.t_begin;
          for (int j = 0; j < nl; ++j) mbar_wait(&tfull[j], 0);
          tc_fence_after();
          mbar_wait(pre_full, 0);
          // (lanes past the tile's columns read column 0: in bounds, never stored)
          const float4* pre = reinterpret_cast<const float4*>(sPre + (lane_ok ? q * LPQ + lane : 0) * MT + h0);
#pragma unroll
          for (int m = 0; m < TPW; m += 4) {
            const float4 v = pre[m / 4];
            g[m] = v.x;
            g[m + 1] = v.y;
            g[m + 2] = v.z;
            g[m + 3] = v.w;
          }
#pragma unroll
          for (int j = 0; j < NACC; ++j) {
            if (j < nl) {
              uint32_t r[NCH][16];
#pragma unroll
              for (int c = 0; c < NCH; ++c) tmem_ld16r(lane_base + j * MT + c * 16, r[c]);
#pragma unroll
              for (int c = 0; c < NCH; ++c) tmem_wait_ld16_dep(r[c]);
#pragma unroll
              for (int c = 0; c < NCH; ++c)
#pragma unroll
                for (int i = 0; i < 16; ++i) g[c * 16 + i] = __fadd_rn(g[c * 16 + i], __uint_as_float(r[c][i]));
            }
          }
          if (lane_ok && n < p.N) {
            const int mlim = p.M - h0;
            float* dst = p.out + static_cast<size_t>(h0) * p.ldo + n;
#pragma unroll
            for (int m = 0; m < TPW; ++m) {
              if (m < mlim) *dst = g[m];
              dst += p.ldo;
            }
          }
          continue;
        }
      }
      int t_in_group = 0;
      uint32_t groups_done = 0;
      for (int t = it.t_begin; t < it.t_end; ++t, ++acc_iter) {
        const int buf = acc_iter % NACC;
        const uint32_t use = acc_iter / NACC;
        mbar_wait(&tfull[buf], use & 1);
        tc_fence_after();
        uint32_t r[NCH][16];
#pragma unroll
        for (int c = 0; c < NCH; ++c) tmem_ld16r(lane_base + buf * MT + c * 16, r[c]);
#pragma unroll
        for (int c = 0; c < NCH; ++c) tmem_wait_ld16_dep(r[c]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        // level 0 (0 + P canonicalises a -0 leaf, matmul.cpp:101-103)
        if (t_in_group == 0 || p.tiles_per_unit == 1) {
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int i = 0; i < 16; ++i) g[c * 16 + i] = __fadd_rn(0.0f, __uint_as_float(r[c][i]));
        } else {
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int i = 0; i < 16; ++i) g[c * 16 + i] = __fadd_rn(g[c * 16 + i], __uint_as_float(r[c][i]));
        }
        if (p.tiles_per_unit > 1 && ++t_in_group < p.kf) continue;
        t_in_group = 0;
        // binary counter over this unit's groups, levels in TMEM slots
        if (p.levels >= 1) {
          int level = 1;
          uint32_t c_bits = groups_done++;
          while (c_bits & 1u) {
            const uint32_t slot = lane_base + (NACC + level - 1) * MT;
#pragma unroll
            for (int c = 0; c < NCH; ++c) tmem_ld16r(slot + c * 16, r[c]);
#pragma unroll
            for (int c = 0; c < NCH; ++c) tmem_wait_ld16_dep(r[c]);
#pragma unroll
            for (int c = 0; c < NCH; ++c)
#pragma unroll
              for (int i = 0; i < 16; ++i) g[c * 16 + i] = __fadd_rn(g[c * 16 + i], __uint_as_float(r[c][i]));
            c_bits >>= 1;
            ++level;
          }
          if (level <= p.levels) {
            const uint32_t slot = lane_base + (NACC + level - 1) * MT;
#pragma unroll
            for (int c = 0; c < NCH; ++c) tmem_st16(slot + c * 16, g + c * 16);
            tmem_wait_st();
            continue;
          }
        }
      }
      // g: this unit's value for column n, tokens h0 .. h0 + TPW - 1
      if (warp == 4 && lane == 0) SK_TRACE(6);
      if (sk_pair_ok<MT, BNW>() && p.pair == 2 && it.unit == 1) {
        // Pair mode 2, finishing CTA: the tile is the two-leaf tree of the units'
        // subtree values, (0 + v1) + (0 + v0) -- the cluster finish's order.
        mbar_wait(pre_full, 0);
        const float4* pre = reinterpret_cast<const float4*>(sPre + (lane_ok ? q * LPQ + lane : 0) * MT + h0);
#pragma unroll
        for (int m = 0; m < TPW; m += 4) {
          const float4 v = pre[m / 4];
          g[m] = __fadd_rn(__fadd_rn(0.0f, g[m]), __fadd_rn(0.0f, v.x));
          g[m + 1] = __fadd_rn(__fadd_rn(0.0f, g[m + 1]), __fadd_rn(0.0f, v.y));
          g[m + 2] = __fadd_rn(__fadd_rn(0.0f, g[m + 2]), __fadd_rn(0.0f, v.z));
          g[m + 3] = __fadd_rn(__fadd_rn(0.0f, g[m + 3]), __fadd_rn(0.0f, v.w));
        }
        if (lane_ok && n < p.N) {
          const int mlim = p.M - h0;
          float* dst = p.out + static_cast<size_t>(h0) * p.ldo + n;
#pragma unroll
          for (int m = 0; m < TPW; ++m) {
            if (m < mlim) *dst = g[m];
            dst += p.ldo;
          }
        }
      } else if (sk_pair_ok<MT, BNW>() && p.pair) {
        // Pair mode, leading CTA: g is its value (mode 1: the prefix fold of the
        // group's first leaves; mode 2: its subtree); hand it to the partner
        // ([column][token] f32) with asynchronous remote stores that complete on
        // the partner's barrier -- no cluster barrier.
        asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
        if (lane_ok) {
          const uint32_t dst =
              dsmem_map(smem_u32(sPre) + static_cast<uint32_t>(((q * LPQ + lane) * MT + h0) * 4), (blockIdx.x & 1u) ^ 1u);
          const uint32_t bar = dsmem_map(smem_u32(pre_full), (blockIdx.x & 1u) ^ 1u);
#pragma unroll
          for (int m = 0; m < TPW; m += 4)
            asm volatile(
                "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                    dst + m * 4),
                "r"(__float_as_uint(g[m])), "r"(__float_as_uint(g[m + 1])), "r"(__float_as_uint(g[m + 2])),
                "r"(__float_as_uint(g[m + 3])), "r"(bar)
                : "memory");
        }
      } else if (p.units == 1) {
        // Straight-line code that runs once per tile: each store is a predicate, a
        // store and a pointer bump (the tail's instructions are fetched cold, so
        // their count is what costs: ~14 per store with per-token index math).
        if (lane_ok && n < p.N) {
          const int mlim = p.M - h0;
          float* dst = p.out + static_cast<size_t>(h0) * p.ldo + n;
#pragma unroll
          for (int m = 0; m < TPW; ++m) {
            if (m < mlim) *dst = g[m];
            dst += p.ldo;
          }
        }
      } else {
        // cluster mode (one item per CTA): publish the unit value in shared memory
        // ([MT][128] f32; every MMA that read the stages has completed)
        float* fbuf = reinterpret_cast<float*>(sW);
#pragma unroll
        if (lane_ok)
#pragma unroll
          for (int m = 0; m < TPW; ++m) fbuf[(h0 + m) * BNW + q * LPQ + lane] = g[m];
      }
    }
  }

  // Finish of a K-split tile inside its cluster: CTA u of the cluster (= unit u)
  // evaluates rows [u R, u R + R) of the tile over all units' values, read from
  // the peers' shared memory (DSMEM):
  //   group j = ((0 + v_{j*fold}) + v_{j*fold+1}) + ...   (level-0 fold; fold = 1
  //             for subtree units, k_first for leaf units)
  //   result  = contiguous-halves tree over the groups (binary counter, new + old)
  // -- the order of tree_combine_kernel (tbik_tree.cu) and of the reference.
  if (warp == 4 && lane == 0) SK_TRACE(7);
  // (a lone CTA needs no cluster barrier: its release fence waits for every
  // outstanding global store, ~1000 cycles)
  if (p.units > 1 && !p.pair) cluster_sync_all();
  if (threadIdx.x == 0) SK_TRACE(8);
  if (p.pair) {
  } else if (p.units == 2) sk_finish<2, BNW>(p, sW);
  else if (p.units == 4) sk_finish<4, BNW>(p, sW);
  else if (p.units == 8) sk_finish<8, BNW>(p, sW);
  else if (p.units > 1) sk_finish<0, BNW>(p, sW);
  if (p.units > 1 && !p.pair) cluster_sync_all();  // peers may still read this CTA's shared memory
  if (threadIdx.x == 0) SK_TRACE(9);
#undef SK_TRACE

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, SK_TMEM_COLS);
  }
}


struct SkKernel {
  void (*kern)(const CUtensorMap, const CUtensorMap, const SkParams);
  size_t smem;
  int threads;
};
template <int MT, int BNW, int KS>
SkKernel sk_entry() {
  return SkKernel{tc_skinny_kernel<MT, BNW, KS>, sk_smem<MT, BNW, KS>(), sk_threads<MT>()};
}
template <int BNW, int KS>
SkKernel sk_select_mt(int mt) {
  static_assert(sk_stages<128, BNW, KS>() >= 3, "skinny stages");
  return mt == 16 ? sk_entry<16, BNW, KS>() : mt == 32 ? sk_entry<32, BNW, KS>()
       : mt == 64 ? sk_entry<64, BNW, KS>() : sk_entry<128, BNW, KS>();
}
SkKernel sk_select(int mt, int bn, int ks) {
  if (bn == 128) return ks == 128 ? sk_select_mt<128, 128>(mt) : sk_select_mt<128, 64>(mt);
  if (bn == 32) return ks == 128 ? sk_select_mt<32, 128>(mt) : sk_select_mt<32, 64>(mt);
  return ks == 128 ? sk_select_mt<64, 128>(mt) : sk_select_mt<64, 64>(mt);
}

}  // namespace

// The skinny variant serves M <= 128 bf16 views (knob tc_skinny = 0 turns it off,
// a pure scheduling choice: the same bits).
bool tc_use_skinny(const GemmView& v) {
  if (knob(KNOB_TC_SKINNY, 1) == 0) return false;
  return v.adt == TBIK_BF16 && v.bdt == TBIK_BF16 && v.M >= 1 && v.M <= SK_MAX_M && v.bk % SK_KSTAGE == 0 &&
         v.N <= (int64_t{1} << 30) && v.K <= (int64_t{1} << 30);
}

tbik_status launch_tc_skinny(const GemmView& v_in, float* C, int64_t ldc, cudaStream_t s) {
  GemmView v = v_in;
  int mt = v.M <= 16 ? 16 : v.M <= 32 ? 32 : v.M <= 64 ? 64 : 128;
  const int force_mt = static_cast<int>(knob(KNOB_SK_MT, 0));  // tuning knob: a wider token tile (same bits)
  if ((force_mt == 32 || force_mt == 64 || force_mt == 128) && force_mt >= mt) mt = force_mt;
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

  SkParams p{};
  p.M = static_cast<int>(v.M);
  p.N = static_cast<int>(v.N);
  p.K = static_cast<int>(v.K);
  p.bk = static_cast<int>(v.bk);
  p.kf = static_cast<int>(v.kf);
  p.T = static_cast<int>(v.T);
  p.out = C;
  p.ldo = ldc;
  // Diagnostics (schedule knob sk_trace = 1): per-CTA phase clocks, their means
  // printed to stderr after each call (synchronises the stream).
  const bool trace = knob(KNOB_SK_TRACE, 0) != 0;
  static unsigned long long* trace_buf = nullptr;
  if (trace && !trace_buf && cudaMalloc(&trace_buf, 4096 * 16 * 8) != cudaSuccess) trace_buf = nullptr;
  p.trace = trace ? trace_buf : nullptr;
  const int64_t want = static_cast<int64_t>(sms) * 7 / 8;
  // Tile width: 64-column tiles (MMA M = 64) when 128-column tiles cover at most
  // half the SMs even with the deepest K split -- short K (TP shards) at decode
  // sizes (measured, tools/decode_bench.py: TP=4 shard M >= 64 -11..16 %, TP=8
  // -2..5 %; TP=1/2 stay faster with 128 columns and K units).
  // (32-column tiles -- MMA M = 64 over a repeated 32-column atom -- are a knob
  // only: a CTA's time is its MMA count (~37 cycles per M = 64 MMA however narrow
  // the tile, tools/micro/small_mma.cu), so twice the CTAs did not help the TP = 8
  // shard: 6.9 vs 6.7 us.)
  const int64_t kunits = std::min<int64_t>(v.L, SK_MAX_UNITS);
  int bn = (v.N + SK_BN - 1) / SK_BN * kunits <= want / 2 ? 64 : SK_BN;
  const int force_bn = static_cast<int>(knob(KNOB_SK_BN, 0));  // tuning knob (same bits)
  if (force_bn == 32 || force_bn == 64 || force_bn == 128) bn = force_bn;
  p.bn = bn;
  p.ntiles = static_cast<int>((v.N + bn - 1) / bn);
  // Units: aligned 2^j-group subtrees (<= 8, one cluster) until the items cover
  // ~7/8 of the SMs (K=14336 N=4096: 4 units, 128 CTAs; measured best vs 2 / 8).
  // Knobs sk_units / sk_leaf override (tuning knobs; same bits).
  const int max_levels = mt == 16 ? sk_max_levels<16>() : mt == 32 ? sk_max_levels<32>()
                       : mt == 64 ? sk_max_levels<64>() : sk_max_levels<128>();
  int64_t units = 1;
  while (units * 2 <= v.L && units * 2 <= SK_MAX_UNITS && p.ntiles * units * 2 <= want) units *= 2;
  const int force_u = static_cast<int>(knob(KNOB_SK_UNITS, 0));
  if (force_u >= 1 && force_u <= v.L && force_u <= SK_MAX_UNITS && (force_u & (force_u - 1)) == 0) units = force_u;
  int lv = 0;
  while ((int64_t{1} << lv) < v.L / units) ++lv;
  if (lv > max_levels) return TBIK_UNSUPPORTED;  // caller falls back to the wide kernel (same bits)
  // Single-leaf units (clusters of T CTAs of one leaf each) measured slower than one
  // unit per tile for the TP=8 down_proj shard (T = 7: 15 vs 9 us at M = 16, CUDA
  // graph; the per-CTA prologue outweighs 64 KB of weights), so they are opt-in.
  const int force_leaf = static_cast<int>(knob(KNOB_SK_LEAF, 0));
  const bool leaf_units = force_leaf != 0 && v.kf > 1 && v.T <= SK_MAX_UNITS;
  if (leaf_units) {
    p.units = static_cast<int>(v.T);
    p.tiles_per_unit = 1;
    p.levels = 0;
    p.fold = static_cast<int>(v.kf);
    int lg = 0;
    while ((int64_t{1} << lg) < v.L) ++lg;
    p.log_groups = lg;
  } else {
    p.units = static_cast<int>(units);
    p.tiles_per_unit = static_cast<int>(v.T / units);
    p.levels = lv;
    p.fold = 1;
    int lg = 0;
    while ((int64_t{1} << lg) < units) ++lg;
    p.log_groups = lg;
  }
  // Pair mode: a tile with a single leaf group (the TP = 8 shard) and no K units
  // runs on two CTAs -- the leading one folds the group's first leaves, the other
  // computes the last <= NACC leaves and continues the fold from the prefix it is
  // sent (same order, same bits).  Each CTA issues about half the small MMAs that
  // bound it (profiles/r02_skinny_decode.md).  Knob sk_pair = 0 turns it off.
  const int nacc = mt >= 128 ? 2 : 4;
  if (knob(KNOB_SK_PAIR, 1) != 0 && !leaf_units && units == 1 && v.L == 1 && mt <= 64 && v.T >= 2 &&
      2 * static_cast<int64_t>(p.ntiles) <= sms) {
    const int t1 = std::min<int>(static_cast<int>(v.T) / 2, nacc);
    p.pair = 1;
    p.units = 2;
    p.tiles_per_unit = static_cast<int>(v.T) - t1;
    p.levels = 0;
    p.fold = 1;
    p.log_groups = 1;
  } else if (knob(KNOB_SK_PAIR, 1) != 0 && !leaf_units && units == 2 && mt <= 32) {
    // two subtree units: the second adds the first's value (no cluster finish);
    // not above 32 tokens, where one CTA storing every row measured slower than
    // the finish split over both (TP = 4 shard M = 64: 11.1 vs 10.8 us)
    p.pair = 2;
  }
  p.items = static_cast<long long>(p.ntiles) * p.units;
  if (p.items >= (int64_t{1} << 31)) return TBIK_UNSUPPORTED;
  TBIK_TRY(pad_operand(&v.A, &v.lda, v.M, v.K, 8, s));
  TBIK_TRY(pad_operand(&v.B, &v.ldb, v.K, v.N, 9, s));
  // K rows per stage: 128 (one 16 KB W box per 64 columns) whenever the leaf is a
  // multiple of 128; knob sk_ks = 64 restores 64-row boxes (same bits: the MMA
  // sequence per leaf is unchanged).
  int ks = v.bk % 128 == 0 ? 128 : 64;
  const int force_ks = static_cast<int>(knob(KNOB_SK_KS, 0));
  if (force_ks == 64 || (force_ks == 128 && v.bk % 128 == 0)) ks = force_ks;
  CUtensorMap mW, mX;
  if (bn == 32)
    TBIK_TRY(tc_make_map_2d_sw64(&mW, v.B, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.K),
                                 static_cast<uint64_t>(v.ldb) * 2, 32, static_cast<uint32_t>(ks)));
  else
    TBIK_TRY(tc_make_map_2d(&mW, v.B, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.K),
                            static_cast<uint64_t>(v.ldb) * 2, 64, static_cast<uint32_t>(ks)));
  TBIK_TRY(tc_make_map_2d(&mX, v.A, static_cast<uint64_t>(v.K), static_cast<uint64_t>(v.M),
                          static_cast<uint64_t>(v.lda) * 2, SK_KSTAGE, static_cast<uint32_t>(mt)));
  const SkKernel sel = sk_select(mt, bn, ks);
  static bool attr_set[16][4][3][2] = {};
  const int mi = mt == 16 ? 0 : mt == 32 ? 1 : mt == 64 ? 2 : 3, bi = bn == 128 ? 2 : bn == 64 ? 1 : 0,
            ki = ks == 128 ? 1 : 0;
  if (dev >= 0 && dev < 16 && !attr_set[dev][mi][bi][ki]) {
    TBIK_CUDA(cudaFuncSetAttribute(sel.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sel.smem)));
    attr_set[dev][mi][bi][ki] = true;
  }
  const size_t smem = sel.smem;
  const int threads = sel.threads;
  const auto kern = sel.kern;
  // X = 1: persistent over tiles; X > 1: one CTA per (tile, unit), clusters of X.
  const long long grid = p.units > 1 ? p.items : (p.items < sms ? p.items : sms);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(static_cast<unsigned>(grid));
  lc.blockDim = dim3(static_cast<unsigned>(threads));
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(p.units);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // Programmatic dependent launch (knob sk_pdl = 0 turns it off): the prologue
  // overlaps the previous kernel when that kernel triggers its dependents.
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = knob(KNOB_SK_PDL, 1) != 0 ? 2 : 1;
  TBIK_CUDA(cudaLaunchKernelEx(&lc, kern, mW, mX, p));
  TBIK_CUDA(cudaGetLastError());
  count_launch("tc_skinny_kernel");
  if (p.trace && grid <= 4096) {
    std::vector<unsigned long long> h(static_cast<size_t>(grid) * 16);
    TBIK_CUDA(cudaStreamSynchronize(s));
    TBIK_CUDA(cudaMemcpy(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost));
    double mean[16] = {0};
    unsigned long long g_lo = ~0ull, g_hi = 0;
    for (long long b = 0; b < grid; ++b) {
      for (int i = 1; i < 10; ++i) mean[i] += static_cast<double>(h[b * 16 + i]) / static_cast<double>(grid);
      g_lo = std::min(g_lo, h[b * 16 + 15]);
      g_hi = std::max(g_hi, h[b * 16 + 15]);
    }
    std::fprintf(stderr,
                 "sk_trace grid %lld ks %d bn %d mt %d | setup %.0f tma0 %.0f mma0 %.0f tma_end %.0f mma_end %.0f "
                 "merge_end %.0f out_end %.0f csync %.0f exit %.0f clk | CTA start spread %llu ns\n",
                 grid, ks, bn, mt, mean[1], mean[2], mean[4], mean[3], mean[5], mean[6], mean[7], mean[8], mean[9],
                 g_hi - g_lo);
  }
  return TBIK_OK;
}

}  // namespace tbik_b200
