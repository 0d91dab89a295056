// tbik_gemm_tc.cu -- the TENSOR-CORE-LEAF TBIK GEMM for sm_100a (v2).
//
// Persistent, 2-CTA (cta_group::2) kernel.  A CTA pair (one cluster) owns a
// 256 x 128 output tile: CTA rank r holds rows [m0 + 128 r, m0 + 128 r + 128)
// of A in shared memory and columns [n0 + 64 r, n0 + 64 r + 64) of B; the
// leader's single MMA thread issues tcgen05.mma.cta_group::2 (M=256, N=128,
// K=16) that reads both CTAs' operands and writes each CTA's 128 x 128 f32
// accumulator into that CTA's TMEM.  Per CTA and per K=16 step this moves
// 6 KB through shared memory (A 4 KB + B 2 KB) instead of 8 KB for a 1-CTA
// 128 x 128 tile.  Pairs loop over work items (output tile x K unit) with an
// L2-grouped raster (8 M-blocks share one pass over W).
//
// Warp roles per CTA (384 threads, one CTA per SM):
//   warp 0      TMA producer: 6-stage ring of {A 128x64, B 64x64} 128B-swizzled
//               tiles (2SM TMA; completion counted on the leader's barrier)
//   warp 1      (leader CTA) MMA issuer: for every leaf tile, block_k/16 MMAs into
//               a ZEROED TMEM accumulator; two accumulators so leaf t+1 is computed
//               while leaf t is merged
//   warp 2      TMEM allocator (512 columns, cta_group::2)
//   warps 4-11  merge warps: warp w may read TMEM lanes 32(w%4)..; thread (w, lane)
//               owns output row 32(w%4) + lane, columns 64((w-4)/4) + [0, 64).
//               For every leaf: both tcgen05.ld chunks in flight, one wait, the
//               accumulator is released, then __fadd_rn verbatim the reference's
//               reduction (k_first == 1: tree level 1 is formed in registers --
//               an even group waits there for its odd sibling):
//                 level 0   g = ((0 + P_0) + P_1) + ... + P_{kf-1}   (matmul.cpp:100-125)
//                 levels>=1 binary counter over group values (matmul.cpp:107-123)
//               g in 64 registers; tree levels 1-2 in TMEM cols [256,512),
//               level 3 in an 8 KB shared-memory region per warp (also the
//               output staging), deeper levels (touched once per 16+ groups) in
//               L2-resident scratch ([col/4][row][4] slabs, 512 B per warp
//               access).  k_first == 1 shifts this up by one: level 1 in
//               registers, 2-3 in TMEM, 4 in shared memory, 5+ in scratch.
//               Results leave through 128B-swizzled 32 x 32 smem boxes and TMA
//               stores.
//   Measured (profiles/r01_tc_merge_ablation*.txt): an L2 round trip for a
//   scratch level stalls the merge for longer than the accumulator double
//   buffer can absorb (-20 % at k_first = 1), hence level 3 on chip at the
//   price of 2 pipeline stages (-1..3 % with the merge disabled).
//   Why this shape (measured, tools/ab_epi.py): the MMA operand reads and TMA
//   writes keep the SM's shared-memory/L1 data port ~90% busy, so every byte the
//   merge moves through L1 costs tensor throughput.  Row-per-thread STG.128
//   costs 32 wavefronts per 512 B; the TMA store path ~4x fewer (+5% at
//   k_first = 1), and 8 merge warps another +6%.
// The arithmetic above the leaf is bit-identical to the reference; the leaf is
// the tensor core's block_k-long accumulation.  Nothing in
// the per-element arithmetic depends on M, the tile position, the unit split, the
// raster or the TP shard -> batch- and TP-invariant by construction.
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>

#include "tbik_common.cuh"
#include "tbik_internal.h"
#include "tbik_mathfn.cuh"
#include "tbik_pair.cuh"

namespace tbik_b200 {

namespace {

using namespace pair_ptx;

constexpr int BM = 128;     // rows per CTA (the pair covers 256)
constexpr int PAIR_M = 256;
constexpr int BN = 128;     // columns per pair tile (MMA N); each CTA stages BN/2 of B
constexpr int KSTAGE = 64;  // K per pipeline stage (one 128 B swizzle row of bf16)
constexpr int STAGES = 6;
constexpr int A_STAGE_BYTES = BM * KSTAGE * 2;        // 16 KB
constexpr int B_STAGE_BYTES = KSTAGE * (BN / 2) * 2;  // 8 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int TMEM_COLS = 512;
constexpr int SLOT_LVL1 = 256;
constexpr int SLOT_LVL2 = 384;
constexpr int GROUP_M = 8;  // raster: M-blocks that share one pass over W
constexpr uint32_t IDESC = umma_idesc_bf16(PAIR_M, BN, /*a_mn_major=*/0, /*b_mn_major=*/1);
constexpr uint32_t IDESC_1CTA = umma_idesc_bf16(BM, BN, /*a_mn_major=*/0, /*b_mn_major=*/1);
// Tree level 3 lives in shared memory: per merge warp an 8 KB region holding its
// 32 rows x 64 columns as [16 float4 columns][32 lanes][float4] (conflict-free
// 16-byte accesses).  The same region doubles as the warp's output staging for
// the TMA store (two 32 x 32 f32 boxes, 128B-swizzled): level 3 is consumed by
// the carry that produces the output, and rewritten only 4+ groups later.
constexpr int OUT_BUF_BYTES = 32 * 32 * 4;
constexpr int L3_WARP_BYTES = 32 * 64 * 4;
// Small-M variants stage only ABOX (< 128) rows of A per stage: the MMA still reads
// a 128-row A window, so consecutive stages' A windows overlap (stride ABOX x 128 B)
// and rows >= ABOX of a window are another stage's bytes -- they only feed output
// rows >= M, which are never stored.  The freed shared memory buys pipeline depth
// for weight streaming (12 stages at ABOX = 32, 9 at 64, 6 at 128).
// Single-CTA variants (PAIR = false, for M <= 128): a CTA owns a 128 x 128 tile
// alone (tcgen05.mma.cta_group::1, M = 128) and stages all 128 columns of B (two
// 64-column atoms) -- half the MMA work per weight column of the pair tile, whose
// second 128 rows would be padding at small M.
constexpr int b_stage_bytes(bool pair) { return pair ? B_STAGE_BYTES : 2 * B_STAGE_BYTES; }
constexpr int a_region_bytes(int abox, int nst) { return (nst - 1) * abox * 128 + A_STAGE_BYTES; }
// DEEP: no shared-memory tree level 3 (it moves to scratch) and a single 4 KB
// output staging box per merge warp; the 32 KB freed per warp pair buys pipeline
// stages.  Free when a work item has <= 2 tree levels (K split into units, TP
// shards, short K) -- the default then; with 3+ levels the on-chip level 3 wins
// (measured, profiles/r01_tc_deep_vs_l3smem.txt).
constexpr int stages_for(int abox, bool pair, bool deep = false) {
  return deep ? (pair ? (abox == 32 ? 15 : abox == 64 ? 11 : 8) : (abox == 32 ? 9 : abox == 64 ? 7 : 6))
              : (pair ? (abox == 32 ? 12 : abox == 64 ? 9 : STAGES) : (abox == 32 ? 7 : abox == 64 ? 6 : 4));
}
// Per merge warp: level-3 slab (32 rows x its 64 columns) that doubles as output
// staging (DEEP: one 4 KB staging box only).
constexpr int MERGE_WARPS = 8;
constexpr int warp_region_bytes(bool deep) { return deep ? OUT_BUF_BYTES : L3_WARP_BYTES; }
constexpr size_t smem_bytes(int abox, bool pair, bool deep = false) {
  return 1024 + static_cast<size_t>(a_region_bytes(abox, stages_for(abox, pair, deep))) +
         static_cast<size_t>(stages_for(abox, pair, deep)) * b_stage_bytes(pair) + 1024 +
         static_cast<size_t>(MERGE_WARPS) * warp_region_bytes(deep);
}
static_assert(smem_bytes(32, true) <= 232448 && smem_bytes(64, true) <= 232448 && smem_bytes(128, true) <= 232448 &&
                  smem_bytes(32, false) <= 232448 && smem_bytes(64, false) <= 232448 &&
                  smem_bytes(128, false) <= 232448 && smem_bytes(32, true, true) <= 232448 &&
                  smem_bytes(64, true, true) <= 232448 && smem_bytes(128, true, true) <= 232448 &&
                  smem_bytes(32, false, true) <= 232448 && smem_bytes(64, false, true) <= 232448 &&
                  smem_bytes(128, false, true) <= 232448,
              "shared memory budget");

struct TcParams {
  int M, N, K;
  int bk, kf, T;
  int tiles_per_unit;
  int units;
  int mode;    // OUT_FULL / OUT_UNITS / OUT_LEAVES
  int levels;  // log2(groups per unit)
  int mblocks, ntiles;
  int tile_m;  // rows per work item: 256 (CTA pair) or 128 (single CTA)
  long long items;
  float* out;
  long long ldo;
  long long unit_stride;
  float* scratch;  // [gridDim.x][levels-3][BN][BM] when levels > 3
  int tma_store;   // 1: results leave through tmC (TMA), 0: direct row stores
  int group_m;     // raster: M-blocks that share one pass over W
  int acc4;        // 1: four TMEM accumulators (items without tree levels leave cols 256-511 free)
  uint16_t* act;   // non-null: SiLU*up epilogue -- columns interleave gate (even) / up (odd);
  long long ld_act;  //   act[row][j] = bf16(silu(g[2j]) * g[2j+1]) replaces the f32 store
  float2* ms_out;  // non-null (FULL mode): also the log-softmax (m, s) state of every 16-column
  long long ld_ms; //   chunk (tb_ms_chunk16): ms_out[row][col / 16] -- the lm_head epilogue
  // Fused tree all-reduce (ar_W > 1; FULL mode, pair tiles): owner(item) = item % ar_W.
  int ar_W, ar_rank;
  uint32_t ar_epoch;
  const float* ar_src[8];
  float* ar_dst[8];
  uint32_t* ar_flags[8];
  uint32_t* ar_done[8];
  uint32_t* ar_counter;
};

struct Item {
  int m0, n0, unit, t_begin, t_end;
};

__device__ __forceinline__ Item decode(const TcParams& p, long long item) {
  Item it;
  it.unit = static_cast<int>(item % p.units);
  const long long rest = item / p.units;
  const int group_m = p.group_m;
  const long long group = group_m * static_cast<long long>(p.ntiles);
  const int g = static_cast<int>(rest / group);
  const int idx = static_cast<int>(rest % group);
  const int gm = min(group_m, p.mblocks - g * group_m);
  const int mb = g * group_m + idx % gm;
  const int nt = idx / gm;
  it.m0 = mb * p.tile_m;
  it.n0 = nt * BN;
  it.t_begin = it.unit * p.tiles_per_unit;
  it.t_end = min(p.T, it.t_begin + p.tiles_per_unit);
  return it;
}

__device__ __forceinline__ int tile_chunks(const TcParams& p, int t) {
  const int kt0 = t * p.bk;
  const int kh = (kt0 + p.bk <= p.K) ? p.bk : p.K - kt0;
  return (kh + KSTAGE - 1) / KSTAGE;
}

// Publish "my half of item `item` is in my send slot" to the item's owner rank:
// flags[owner][(item * 2 + cta) * W + my_rank] = epoch.
__device__ __forceinline__ void ar_publish(const TcParams& p, long long item, uint32_t cta) {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __threadfence_system();
  const int owner = static_cast<int>(item % p.ar_W);
  st_release_sys(p.ar_flags[owner] + ((item * 2 + cta) * p.ar_W + p.ar_rank), p.ar_epoch);
}

// Fused all-reduce of ONE owned item's 128-row half (this CTA's), by threads
// rt = 0..nthr-1 meeting on named barrier `bar_id`: wait for the W ranks' tile
// flags, reduce in Algorithm-2 order (collective.cpp:67-74) from the peers' send
// slots, push the result into every rank's result slot.
__device__ __forceinline__ void ar_reduce_item(const TcParams& p, long long item, uint32_t rank, int rt, int nthr,
                                               int bar_id) {
  const int W = p.ar_W;
  const Item it = decode(p, item);
  if (rt < W) spin_until_epoch(p.ar_flags[p.ar_rank] + ((item * 2 + rank) * W + rt), p.ar_epoch);
  named_bar(bar_id, nthr);
  const int r0 = it.m0 + static_cast<int>(rank) * BM;
  const int rows = min(BM, p.M - r0);
  const int cols = min(BN, p.N - it.n0);
  if (rows <= 0) return;
  if (cols == BN && (p.ldo & 3) == 0) {
    // 2 float4 per thread per round, all W loads of the round in flight at once
    // (NVLink latency-bound with few warps: the ILP matters); L2-only loads -- the
    // flag acquire + barrier above order them after the peers' stores.
    constexpr int U = 2;
    const int nq = rows * (BN / 4);
    for (int base = 0; base < nq; base += nthr * U) {
      size_t e4[U];
      float4 r[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * nthr + rt;
        e4[u] = idx < nq ? (static_cast<size_t>(r0 + idx / (BN / 4)) * p.ldo + it.n0) / 4 + idx % (BN / 4) : 0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < W && idx < nq) r[u][k] = __ldcg(reinterpret_cast<const float4*>(p.ar_src[k]) + e4[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (base + u * nthr + rt >= nq) continue;
#pragma unroll
        for (int l = 1; l <= 3; ++l) {
          const int st = 1 << l, h = 1 << (l - 1);
#pragma unroll
          for (int left = 0; left < 8; left += st)
            if (left + h < W) {
              r[u][left].x = __fadd_rn(r[u][left].x, r[u][left + h].x);
              r[u][left].y = __fadd_rn(r[u][left].y, r[u][left + h].y);
              r[u][left].z = __fadd_rn(r[u][left].z, r[u][left + h].z);
              r[u][left].w = __fadd_rn(r[u][left].w, r[u][left + h].w);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < W) reinterpret_cast<float4*>(p.ar_dst[(p.ar_rank + k) & (W - 1)])[e4[u]] = r[u][0];
      }
    }
  } else {
    const int ne = rows * cols;
    for (int idx = rt; idx < ne; idx += nthr) {
      const size_t e = static_cast<size_t>(r0 + idx / cols) * p.ldo + it.n0 + idx % cols;
      float r[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < W) r[k] = __ldcv(p.ar_src[k] + e);
#pragma unroll
      for (int l = 1; l <= 3; ++l) {
        const int st = 1 << l, h = 1 << (l - 1);
#pragma unroll
        for (int left = 0; left < 8; left += st)
          if (left + h < W) r[left] = __fadd_rn(r[left], r[left + h]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < W) p.ar_dst[(p.ar_rank + k) & (W - 1)][e] = r[0];
    }
  }
  }

// Warps 2-3 during the GEMM: every owned item of this pair except the pair's last
// one, which all warps reduce together once the GEMM loops are done (the kernel's
// tail would otherwise wait on two warps' NVLink loads).
__device__ __forceinline__ void ar_reduce_owned(const TcParams& p, long long pair, long long npairs, uint32_t rank) {
  const long long last = pair < p.items ? pair + (p.items - 1 - pair) / npairs * npairs : -1;
  for (long long item = pair; item < p.items; item += npairs)
    if (item != last && static_cast<int>(item % p.ar_W) == p.ar_rank)
      ar_reduce_item(p, item, rank, static_cast<int>(threadIdx.x) - 64, 64, 2);
}

// After the GEMM loops, all threads of the CTA: the pair's last item if owned, then
// (every CTA of this rank done) the last CTA publishes done[rank] to all peers.
__device__ __forceinline__ void ar_finish(const TcParams& p, long long pair, long long npairs, uint32_t rank) {
  const long long last = pair < p.items ? pair + (p.items - 1 - pair) / npairs * npairs : -1;
  if (last >= 0 && static_cast<int>(last % p.ar_W) == p.ar_rank)
    ar_reduce_item(p, last, rank, static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x), 3);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(p.ar_counter, 1u);
    if (prev == gridDim.x - 1) {
      *p.ar_counter = 0;
      __threadfence_system();
      for (int r = 0; r < p.ar_W; ++r) st_release_sys(p.ar_done[r] + p.ar_rank, p.ar_epoch);
    }
  }
}


// EPI = 8 merge warps (two per TMEM lane quarter, splitting the 128 columns).
// ABOX A rows staged per stage (128, or 64 / 32 for small M; stage count follows).
// KF1 (used when k_first == 1, where every leaf completes a group): tree level 1
// never touches TMEM -- an even group stays in registers and the odd sibling
// merges into it, so a pair of leaves costs two accumulator drains instead of two
// drains + a level-1 store + load.
// AR: the fused tree all-reduce variant (pair tiles, FULL mode; tbik_group.cu).
// MSE: the lm_head variant -- the epilogue also emits the log-softmax (m, s) state
// of every 16-column chunk (a separate instantiation: the exp code would otherwise
// cost the plain GEMM registers).
constexpr int EPI = MERGE_WARPS;
template <bool KF1, int ABOX, bool PAIR, bool DEEP, bool AR = false, bool MSE = false>
__global__ void __launch_bounds__(128 + 32 * EPI, 1)
    tc_tree_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC, const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  constexpr int NST = stages_for(ABOX, PAIR, DEEP);
  constexpr int A_STRIDE = ABOX * 128;  // bytes between consecutive stages' A windows
  constexpr int B_STAGE = b_stage_bytes(PAIR);
  constexpr uint32_t TX_BYTES = A_STRIDE + B_STAGE;
  uint8_t* sB = smem + a_region_bytes(ABOX, NST);
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + NST * B_STAGE);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  // Two TMEM accumulators, or four when the items carry no tree level (one leaf
  // group per item: TP shards) -- the level slots' columns [256, 512) are free
  // then, and the MMA may run up to three leaves ahead of the output epilogue.
  uint64_t* tempty = tfull + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  uint8_t* sL3 = sB + NST * B_STAGE + 1024;  // 1024-aligned level-3 / output staging

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = PAIR ? cluster_rank() : 0;
  const uint32_t rank = crank & 1;  // rank within the CTA pair
  const uint32_t leader_rank = crank & ~1u;
  const bool leader = rank == 0;
  const long long pair = PAIR ? blockIdx.x >> 1 : blockIdx.x;  // work-item stream
  const long long npairs = PAIR ? gridDim.x >> 1 : gridDim.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], PAIR ? 2 : 1);  // one arrive.expect_tx per CTA (leader's copy used)
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&tfull[b], 1);   // multicast commit
      mbar_init(&tempty[b], PAIR ? 2 * EPI : EPI);  // EPI merge warps per CTA (leader's copy used)
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR)
      tmem_alloc_2cta(tmem_slot, TMEM_COLS);
    else
      tmem_alloc(tmem_slot, TMEM_COLS);
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch (knob tc_pdl; not for the fused all-reduce form):
  // operands, scratch and output are touched only after the previous kernel has
  // completed; dependents may launch once every CTA got here.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");

  if (warp < 4) {
  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (elect_one()) {
      const uint32_t full_leader0 = mapa(smem_u32(&full[0]), leader_rank);
      int stage = 0;
      uint32_t phase = 0;
      for (long long item = pair; item < p.items; item += npairs) {
        const Item it = decode(p, item);
        const int am = it.m0 + static_cast<int>(rank) * BM;
        const int bn = it.n0 + static_cast<int>(rank) * (BN / 2);
        for (int t = it.t_begin; t < it.t_end; ++t) {
          const int nch = tile_chunks(p, t);
          for (int c = 0; c < nch; ++c) {
            mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t fb = full_leader0 + stage * 8;
            if (leader)
              mbar_arrive_expect_tx(&full[stage], TX_BYTES);
            else
              mbar_arrive_expect_tx_cluster(fb, TX_BYTES);
            const int k = t * p.bk + c * KSTAGE;
            if constexpr (PAIR) {
              tma_load_2d_2sm(sA + stage * A_STRIDE, &tmA, fb, k, am);
              tma_load_2d_2sm(sB + stage * B_STAGE, &tmB, fb, bn, k);
            } else {  // all 128 columns: two 64-column atoms
              tma_load_2d(sA + stage * A_STRIDE, &tmA, &full[stage], k, am);
              tma_load_2d(sB + stage * B_STAGE, &tmB, &full[stage], bn, k);
              tma_load_2d(sB + stage * B_STAGE + B_STAGE_BYTES, &tmB, &full[stage], bn + BN / 2, k);
            }
            if (++stage == NST) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    // The whole warp runs the loop (its control values are warp-uniform, so they
    // live in uniform registers) and one elected lane issues.  Descriptors are
    // built once and advanced by constant offsets: round 1's per-MMA descriptor
    // arithmetic -- ~90 dependent instructions per 64-K stage on a single thread
    // -- kept the MMA issuer, not the operand feed, on the critical path
    // (ncu source-level samples, profiles/r02_ncu_mma_issuer.md).
    if (leader) {
      // SW128 descriptors (umma_desc_sw128): lo = start >> 4 | LBO >> 4 << 16, hi =
      // SBO >> 4 | version bit 46 | layout SWIZZLE_128B (bits 61-63).  Shared
      // addresses stay below 2^18, so the 14-bit start field never carries.
      constexpr uint32_t DESC_HI = (1024u >> 4) | (1u << 14) | (2u << 29);
      const uint32_t a_lo0 = (smem_u32(sA) >> 4) | ((16u >> 4) << 16);                 // A: K-major
      const uint32_t b_lo0 = (smem_u32(sB) >> 4) | ((uint32_t(B_STAGE_BYTES) >> 4) << 16);  // B: MN-major
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc_iter = 0;
      for (long long item = pair; item < p.items; item += npairs) {
        const Item it = decode(p, item);
        for (int t = it.t_begin; t < it.t_end; ++t, ++acc_iter) {
          const int buf = p.acc4 ? acc_iter & 3 : acc_iter & 1;
          const uint32_t use = p.acc4 ? acc_iter >> 2 : acc_iter >> 1;
          mbar_wait(&tempty[buf], (use & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + buf * BN;
          const int nch = tile_chunks(p, t);
          for (int c = 0; c < nch; ++c) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a_lo = a_lo0 + static_cast<uint32_t>(stage) * (A_STRIDE >> 4);
            const uint32_t b_lo = b_lo0 + static_cast<uint32_t>(stage) * (B_STAGE >> 4);
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < KSTAGE / 16; ++kk) {
                // A: +32 B per 16-element K step inside the 128 B swizzle atom.
                // B: 64-column atoms B_STAGE_BYTES apart (LBO; one atom per CTA in a
                // pair, two in a single CTA), 8-row K groups 1 KB apart (SBO), +16 K
                // rows (2 KB) per step.
                const uint64_t adesc = (static_cast<uint64_t>(DESC_HI) << 32) | (a_lo + kk * (32 >> 4));
                const uint64_t bdesc = (static_cast<uint64_t>(DESC_HI) << 32) | (b_lo + kk * (2048 >> 4));
                if constexpr (PAIR)
                  umma_bf16_2cta(d, adesc, bdesc, IDESC, (c | kk) != 0 ? 1u : 0u);
                else
                  umma_bf16(d, adesc, bdesc, IDESC_1CTA, (c | kk) != 0 ? 1u : 0u);
              }
              if constexpr (PAIR)
                umma_commit_2cta(&empty[stage], 0x3);
              else
                umma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == NST) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (elect_one()) {
            if constexpr (PAIR)
              umma_commit_2cta(&tfull[buf], static_cast<uint16_t>(0x3u << leader_rank));
            else
              umma_commit(&tfull[buf]);
          }
          __syncwarp();
        }
      }
    }
    __syncwarp();
  } else if (AR) {
    // ---------------- fused tree all-reduce (warps 2-3, both CTAs) ----------------
    // For every item this pair computes and this rank owns (item % W == rank): wait
    // until all W ranks published this CTA's 128-row half of it, reduce it in
    // Algorithm-2 order (collective.cpp:67-74) straight from the peers' send slots
    // and push the result into every rank's result slot over NVLink -- while the
    // tensor cores of the same SM already work on the next items.
    ar_reduce_owned(p, pair, npairs, rank);
  }
  } else {
    // ---------------- merge warps (the TBIK reduction), both CTAs ----------------
    constexpr int COLS = BN * 4 / EPI;  // columns owned by this thread (64)
    constexpr int NCH = COLS / 32;
    const int q = warp & 3;  // a warp may only touch TMEM lanes 32*(warp%4)..
    const int col0 = ((warp - 4) >> 2) * COLS;
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + col0;
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), leader_rank);
    // TMEM holds tree levels 1-2, shared memory level 3 (this warp's sL3 region);
    // levels >= 4 live in scratch as [col/4][row][4] slabs (a warp's float4
    // access is 512 contiguous bytes).
    // k_first == 1 keeps level 1 in registers, so its TMEM columns hold level 3
    // (off the shared-memory port the MMA operand reads saturate); scratch from 4.
    // ... and shared memory (when not DEEP) holds level 4.
    constexpr int SL = KF1 ? 4 : 3;                        // the shared-memory level
    constexpr int FS = DEEP ? SL : SL + 1;                 // first scratch level
    float* scratch_base =
        p.levels >= FS
            ? p.scratch + static_cast<size_t>(blockIdx.x) * static_cast<size_t>(p.levels - FS + 1) * (BM * BN) +
                           static_cast<size_t>(col0) * BM + static_cast<size_t>(row_in_tile) * 4
            : nullptr;
    uint8_t* l3 = sL3 + (warp - 4) * warp_region_bytes(DEEP);  // [COLS/4][32 lanes][float4] (+ staging)
    constexpr bool ONE_BOX = DEEP;  // a single staging box per warp

    float g[COLS];  // level 0: the running leaf-group value
    int xb = 0;      // output staging buffer toggle
    uint32_t acc_iter = 0;
    for (long long item = pair; item < p.items; item += npairs) {
      const Item it = decode(p, item);
      const int grow = it.m0 + static_cast<int>(rank) * BM + row_in_tile;
      const bool row_ok = grow < p.M;
      const int ncols = min(COLS, p.N - it.n0 - col0);
      int t_in_group = 0;
      uint32_t groups_done = 0;
      for (int t = it.t_begin; t < it.t_end; ++t, ++acc_iter) {
        const int buf = p.acc4 ? acc_iter & 3 : acc_iter & 1;
        const uint32_t use = p.acc4 ? acc_iter >> 2 : acc_iter >> 1;
        mbar_wait(&tfull[buf], use & 1);
        tc_fence_after();
        const uint32_t acc = lane_base + buf * BN;
        // Both 32-column chunks in flight at once, one wait (for k_first == 1 on an
        // odd group: each leaf chunk together with the level-1 slot chunk it merges
        // with); the accumulator goes back to the MMA issuer as soon as the values
        // are in registers.
        uint32_t r[NCH < 2 ? 2 : NCH][32];
        const bool odd = KF1 && p.levels >= 1 && (groups_done & 1u);
#pragma unroll
        for (int c = 0; c < NCH; ++c) tmem_ld32r(acc + c * 32, r[c]);
#pragma unroll
        for (int c = 0; c < NCH; ++c) tmem_wait_ld_dep(r[c]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader)
            mbar_arrive(&tempty[buf]);
          else
            mbar_arrive_cluster(tempty_leader0 + buf * 8);
        }
        int unit_out = p.mode == OUT_UNITS ? it.unit : 0;
        if (p.mode == OUT_LEAVES) {
          // verification dump: the raw leaf P_t goes to slice t
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i) g[c * 32 + i] = __uint_as_float(r[c][i]);
          unit_out = t;
        } else {
        // level 0: g = ((0 + P_0) + P_1) + ... + P_{kf-1}   (matmul.cpp:100-125; 0 + P
        // canonicalises a -0 leaf like matmul.cpp:101-103)
        if (odd) {
          // level 1 in registers: g holds the previous group S1 (kept since the even
          // leaf); the new group (0 + P) merges with it, new + old (matmul.cpp:107-123)
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              g[c * 32 + i] = __fadd_rn(__fadd_rn(0.0f, __uint_as_float(r[c][i])), g[c * 32 + i]);
        } else if (KF1 || t_in_group == 0) {  // KF1 <=> k_first == 1: every leaf starts a group
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i) g[c * 32 + i] = __fadd_rn(0.0f, __uint_as_float(r[c][i]));
        } else {
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i) g[c * 32 + i] = __fadd_rn(g[c * 32 + i], __uint_as_float(r[c][i]));
        }
        if (!KF1 && ++t_in_group < p.kf) continue;
        t_in_group = 0;

        // Binary counter over completed groups (levels 1..p.levels, matmul.cpp:107-123):
        // levels 1-2 in TMEM columns [256, 512), deeper levels (touched once per 8+
        // groups) in L2-resident scratch.
        if (KF1 && p.levels >= 1 && !odd) {  // even group: stays in registers as level 1
          ++groups_done;
          continue;
        }
        if (p.levels >= 1) {
          int level = 1;
          uint32_t c_bits = groups_done++;
          if (odd) {  // the level-1 merge happened with the leaf load
            c_bits >>= 1;
            level = 2;
          }
          while (c_bits & 1u) {
            if (KF1 ? (level == 2 || level == 3) : level <= 2) {
              const uint32_t slot = lane_base + (level == 2 ? SLOT_LVL2 : SLOT_LVL1);
#pragma unroll
              for (int c = 0; c < NCH; ++c) tmem_ld32r(slot + c * 32, r[c]);
#pragma unroll
              for (int c = 0; c < NCH; ++c) tmem_wait_ld_dep(r[c]);
#pragma unroll
              for (int c = 0; c < NCH; ++c)
#pragma unroll
                for (int i = 0; i < 32; ++i) g[c * 32 + i] = __fadd_rn(g[c * 32 + i], __uint_as_float(r[c][i]));
            } else if (!DEEP && level == SL) {
#pragma unroll
              for (int i = 0; i < COLS; i += 4) {
                const float4 x = *reinterpret_cast<const float4*>(l3 + ((i / 4) * 32 + lane) * 16);
                g[i] = __fadd_rn(g[i], x.x);
                g[i + 1] = __fadd_rn(g[i + 1], x.y);
                g[i + 2] = __fadd_rn(g[i + 2], x.z);
                g[i + 3] = __fadd_rn(g[i + 3], x.w);
              }
              __syncwarp();  // the region may become output staging right after
            } else {
              const float* sp = scratch_base + static_cast<size_t>(level - FS) * (BM * BN);
#pragma unroll
              for (int i = 0; i < COLS; i += 4) {
                const float4 x = *reinterpret_cast<const float4*>(sp + i * BM);
                g[i] = __fadd_rn(g[i], x.x);
                g[i + 1] = __fadd_rn(g[i + 1], x.y);
                g[i + 2] = __fadd_rn(g[i + 2], x.z);
                g[i + 3] = __fadd_rn(g[i + 3], x.w);
              }
            }
            c_bits >>= 1;
            ++level;
          }
          if (level <= p.levels) {
            if (KF1 ? (level == 2 || level == 3) : level <= 2) {
              const uint32_t slot = lane_base + (level == 2 ? SLOT_LVL2 : SLOT_LVL1);
#pragma unroll
              for (int c = 0; c < NCH; ++c) {
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = g[c * 32 + i];
                tmem_st32(slot + c * 32, v);
              }
              tmem_wait_st();
            } else if (!DEEP && level == SL) {
              if (lane == 0) bulk_wait_read<0>();  // earlier output boxes staged here
              __syncwarp();
#pragma unroll
              for (int i = 0; i < COLS; i += 4)
                *reinterpret_cast<float4*>(l3 + ((i / 4) * 32 + lane) * 16) =
                    make_float4(g[i], g[i + 1], g[i + 2], g[i + 3]);
            } else {
              float* sp = scratch_base + static_cast<size_t>(level - FS) * (BM * BN);
#pragma unroll
              for (int i = 0; i < COLS; i += 4)
                *reinterpret_cast<float4*>(sp + i * BM) = make_float4(g[i], g[i + 1], g[i + 2], g[i + 3]);
            }
            continue;
          }
        }
        }  // the carry left the top level: g is this unit's complete (sub)tree
        if (MSE && row_ok) {
          // lm_head: the (m, s) state of each of this thread's four 16-column chunks,
          // computed on the final f32 logits in registers (F2: the log-softmax's
          // first pass never re-reads the logits from HBM)
#pragma unroll
          for (int j = 0; j < COLS / TB_MS_CHUNK; ++j) {
            const int col = it.n0 + col0 + j * TB_MS_CHUNK;
            if (col < p.N) {
              float v[TB_MS_CHUNK];
#pragma unroll
              for (int i = 0; i < TB_MS_CHUNK; ++i) v[i] = g[j * TB_MS_CHUNK + i];
              float cm, cs;
              tb_ms_chunk16(v, cm, cs);
              p.ms_out[static_cast<size_t>(grow) * p.ld_ms + col / TB_MS_CHUNK] = make_float2(cm, cs);
            }
          }
        }
        if (p.act) {
          // fused SiLU(gate) * up (tb_silu_mul_bf16, the same ops as tbik_silu_mul):
          // this thread's 64 columns are 32 (gate, up) pairs -> 32 bf16 outputs
          if (row_ok) {
            uint16_t* dst = p.act + static_cast<size_t>(grow) * p.ld_act + (it.n0 + col0) / 2;
            const int npair = ncols / 2;
            if (npair == COLS / 2 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
              for (int q8 = 0; q8 < COLS / 16; ++q8) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int c = q8 * 16 + 4 * e;
                  w[e] = static_cast<uint32_t>(tb_silu_mul_bf16(g[c], g[c + 1])) |
                         (static_cast<uint32_t>(tb_silu_mul_bf16(g[c + 2], g[c + 3])) << 16);
                }
                *reinterpret_cast<uint4*>(dst + q8 * 8) = make_uint4(w[0], w[1], w[2], w[3]);
              }
            } else {
#pragma unroll
              for (int jj = 0; jj < COLS / 2; ++jj)
                if (jj < npair) dst[jj] = tb_silu_mul_bf16(g[2 * jj], g[2 * jj + 1]);
            }
          }
        } else if (p.tma_store) {
          // Row-per-lane registers -> 128B-swizzled 32 x 32 smem box (conflict-free
          // 16 B stores) -> one TMA store per box; the tensor map clips ragged edges.
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            if (lane == 0) {
              if constexpr (ONE_BOX)
                bulk_wait_read<0>();  // one staging box per warp
              else
                bulk_wait_read<1>();
            }
            __syncwarp();
            uint8_t* sbuf = l3 + (ONE_BOX ? 0 : xb * OUT_BUF_BYTES);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(sbuf + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                  make_float4(g[c * 32 + 4 * j], g[c * 32 + 4 * j + 1], g[c * 32 + 4 * j + 2], g[c * 32 + 4 * j + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&tmC, smem_u32(sbuf), it.n0 + col0 + c * 32, grow - lane, unit_out);
              bulk_commit();
            }
            xb ^= 1;
          }
        } else if (row_ok) {
          float* dst = p.out + static_cast<size_t>(unit_out) * p.unit_stride + static_cast<size_t>(grow) * p.ldo +
                       it.n0 + col0;
          if (ncols == COLS && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
            for (int i = 0; i < COLS; i += 4)
              *reinterpret_cast<float4*>(dst + i) = make_float4(g[i], g[i + 1], g[i + 2], g[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < COLS; ++i)
              if (i < ncols) dst[i] = g[i];
          }
        }
      }
      if constexpr (AR) {
        // fused all-reduce: the previous item's stores have completed once only this
        // item's NCH store groups may still be pending; publish it to its owner
        if (lane == 0) bulk_wait_complete<NCH>();
        named_bar(1, 32 * EPI);
        if (warp == 4 && lane == 0 && item >= pair + npairs) ar_publish(p, item - npairs, rank);
      }
    }
    if (p.tma_store && lane == 0) bulk_wait_all();
    if constexpr (AR) {
      named_bar(1, 32 * EPI);
      if (warp == 4 && lane == 0 && pair < p.items)  // this pair's last item
        ar_publish(p, pair + (p.items - 1 - pair) / npairs * npairs, rank);
    }
  }

  if constexpr (AR) {
    __syncthreads();  // every role's loop is done (the merge warps published all items)
    ar_finish(p, pair, npairs, rank);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR)
      tmem_dealloc_2cta(tmem_base, TMEM_COLS);
    else
      tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ---- host side ---------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

tbik_status make_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                        uint32_t box_inner, uint32_t box_outer,
                        CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return TBIK_OK;
}

// f32 output [units][M][N] (row stride, unit stride in bytes), 32 x 32 boxes,
// 128B swizzle (matches the merge warps' staging layout).
tbik_status make_map_out(CUtensorMap* map, float* base, uint64_t n, uint64_t m, uint64_t units,
                         uint64_t row_stride_bytes, uint64_t unit_stride_bytes) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {n, m, units};
  cuuint64_t strides[2] = {row_stride_bytes, unit_stride_bytes};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled(out) failed: " + std::to_string(r));
  return TBIK_OK;
}

thread_local int g_sm_cap = 0;  // set_tc_sm_cap: leave SMs free for a concurrent kernel
thread_local FusedAr* g_fused_ar = nullptr;  // set_tc_fused_ar

int sm_count() {
  static int n[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  if (dev >= 0 && dev < 16) {
    if (!n[dev]) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
    if (n[dev]) sms = n[dev];
  }
  return g_sm_cap > 0 && g_sm_cap < sms ? (g_sm_cap & ~1) : sms;
}

}  // namespace

tbik_status tc_make_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  return make_map_2d(map, base, inner, outer, row_stride_bytes, box_inner, box_outer);
}

// 32-byte swizzle (16-column bf16 boxes): the MN-major B atoms of the 256x192 kernel.
// bf16 [1][M][N] output of the SiLU*up epilogue, no swizzle (box rows of box_n
// elements), as a 3D map so the kernels' TMA-store helper serves it unchanged.
tbik_status tc_make_map_act(CUtensorMap* map, uint16_t* base, uint64_t n, uint64_t m, uint64_t row_stride_bytes,
                            uint32_t box_n, uint32_t box_m) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {n, m, 1};
  cuuint64_t strides[2] = {row_stride_bytes, row_stride_bytes * m};
  cuuint32_t box[3] = {box_n, box_m, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled(act) failed: " + std::to_string(r));
  return TBIK_OK;
}

// bf16 3-D map {d0, d1, d2} (d0 contiguous), 128-byte swizzle, box {box0, box1, 1}:
// boxes never cross d2 (out-of-range rows of d1 read as zeros).
tbik_status tc_make_map_3d_bf16_sw128(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled(3d) failed: " + std::to_string(r));
  return TBIK_OK;
}

tbik_status tc_make_map_2d_sw32(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                                uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  return make_map_2d(map, base, inner, outer, row_stride_bytes, box_inner, box_outer, CU_TENSOR_MAP_SWIZZLE_32B);
}

tbik_status tc_make_map_2d_sw64(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                                uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  return make_map_2d(map, base, inner, outer, row_stride_bytes, box_inner, box_outer, CU_TENSOR_MAP_SWIZZLE_64B);
}

tbik_status tc_make_map_out(CUtensorMap* map, float* base, uint64_t n, uint64_t m, uint64_t units,
                            uint64_t row_stride_bytes, uint64_t unit_stride_bytes) {
  return make_map_out(map, base, n, m, units, row_stride_bytes, unit_stride_bytes);
}

FusedAr* set_tc_fused_ar(FusedAr* ctx) {
  FusedAr* old = g_fused_ar;
  g_fused_ar = ctx;
  return old;
}

int set_tc_sm_cap(int cap) {
  const int old = g_sm_cap;
  g_sm_cap = cap;
  return old;
}

bool tc_supported(const GemmView& v, std::string* why) {
  auto no = [&](const char* w) {
    if (why) *why = w;
    return false;
  };
  if (v.adt != TBIK_BF16 || v.bdt != TBIK_BF16) return no("tcgen05 leaf needs bf16 A and B");
  if (v.bk % KSTAGE) return no("tcgen05 leaf needs block_k % 64 == 0");
  if (v.lda % 8 || v.ldb % 8) return no("tcgen05 leaf needs lda, ldb multiples of 8 (16-byte TMA strides)");
  if ((reinterpret_cast<uintptr_t>(v.A) & 15) || (reinterpret_cast<uintptr_t>(v.B) & 15))
    return no("tcgen05 leaf needs 16-byte aligned A and B");
  if (v.M > (1ll << 30) || v.N > (1ll << 30) || v.K > (1ll << 30)) return no("dimension too large");
  return true;
}

// Single-CTA 128 x 128 tiles when every row fits one CTA (M <= 128): the pair
// tile's second 128 rows would be MMA work on padding.  Schedule knob tc_pair
// forces the choice (a pure scheduling knob: same bits).
bool tc_use_pair(const GemmView& v) {
  const int64_t k = knob(KNOB_TC_PAIR, -1);
  if (k == 0 || k == 1) return k == 1;
  return v.M > BM;
}

int64_t tc_pair_tiles(const GemmView& v) { return ((v.M + PAIR_M - 1) / PAIR_M) * ((v.N + BN - 1) / BN); }

int64_t tc_parallel_slots(const GemmView& v) { return tc_use_pair(v) ? sm_count() / 2 : sm_count(); }

int64_t tc_tiles(const GemmView& v) {
  if (tc_use_pair(v)) return tc_pair_tiles(v);
  return ((v.M + BM - 1) / BM) * ((v.N + BN - 1) / BN);
}

// Diagnostics build only (see tools/tc_stats.py); the production kernel carries no counters.
int tc_debug_stats(unsigned long long*, int) { return 0; }

namespace {
// cudaFuncSetAttribute applies to one device context: remembered per (device, kernel).
bool attr_done(int dev, const void* kern) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  std::lock_guard<std::mutex> lk(mu);
  return !done.insert({dev, kern}).second;
}
}  // namespace

tbik_status launch_tc_gemm(const GemmView& v_in, const GemmOut& o, cudaStream_t s) {
  GemmView v = v_in;
  if (v.adt == TBIK_BF16 && v.bdt == TBIK_BF16) {  // any K / N: pad strides for TMA
    TBIK_TRY(pad_operand(&v.A, &v.lda, v.M, v.K, 8, s));
    TBIK_TRY(pad_operand(&v.B, &v.ldb, v.K, v.N, 9, s));
  }
  std::string why;
  if (!tc_supported(v, &why)) return set_error(TBIK_UNSUPPORTED, why);
  if (o.mode == OUT_GROUPS) return set_error(TBIK_BAD_ARGUMENT, "tc gemm: GROUPS mode is FMA-only");
  // 256 x 192 pair tiles (tbik_gemm_tc_w192.cu) for plain FULL / UNITS launches.
  if (!g_fused_ar && tc_use_pair(v) && tc_wide_supported(v, o)) {
    if (tc_wide_variant(v) != 0) {
      const tbik_status st = launch_tc_w192(v, o, s);
      if (st != TBIK_UNSUPPORTED) return st;
    }
  }
  // A rows staged per stage: the fewest that still cover every row of the pair
  // tile's leader CTA (knob tc_abox overrides, a pure scheduling knob).
  int abox = v.M <= 32 ? 32 : v.M <= 64 ? 64 : 128;
  {
    const int64_t a = knob(KNOB_TC_ABOX, 0);
    if ((a == 32 && v.M <= 32) || (a == 64 && v.M <= 64) || a == 128) abox = static_cast<int>(a);
  }
  CUtensorMap mA, mB;
  TBIK_TRY(make_map_2d(&mA, v.A, static_cast<uint64_t>(v.K), static_cast<uint64_t>(v.M),
                       static_cast<uint64_t>(v.lda) * 2, KSTAGE, static_cast<uint32_t>(abox)));
  TBIK_TRY(make_map_2d(&mB, v.B, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.K),
                       static_cast<uint64_t>(v.ldb) * 2, BN / 2, KSTAGE));
  TcParams p{};
  p.M = static_cast<int>(v.M);
  p.N = static_cast<int>(v.N);
  p.K = static_cast<int>(v.K);
  p.bk = static_cast<int>(v.bk);
  p.kf = static_cast<int>(v.kf);
  p.T = static_cast<int>(v.T);
  p.mode = o.mode;
  p.out = o.out;
  p.ldo = o.ldo;
  p.unit_stride = o.unit_stride;
  p.act = o.act;
  p.ld_act = o.ld_act;
  p.ms_out = reinterpret_cast<float2*>(o.ms);
  p.ld_ms = o.ld_ms / 2;
  if (o.ms && (o.mode != OUT_FULL || o.act || (reinterpret_cast<uintptr_t>(o.ms) & 7) || (o.ld_ms & 1)))
    return set_error(TBIK_BAD_ARGUMENT, "tc gemm: chunk (m, s) epilogue needs FULL mode, f32 output, 8-byte states");
  if (o.act && (o.mode != OUT_FULL || v.N % 2)) return set_error(TBIK_BAD_ARGUMENT, "tc gemm: SiLU epilogue needs FULL mode and even N");
  if (o.mode == OUT_LEAVES) {
    p.tiles_per_unit = 1;
    p.levels = 0;
    p.units = p.T;
  } else {
    p.tiles_per_unit = static_cast<int>(o.tiles_per_unit);
    if (p.tiles_per_unit % p.kf) return set_error(TBIK_BAD_ARGUMENT, "tc gemm: unit not whole groups");
    const int64_t groups = p.tiles_per_unit / p.kf;
    if (groups & (groups - 1)) return set_error(TBIK_BAD_ARGUMENT, "tc gemm: unit not 2^j groups");
    int lv = 0;
    while ((int64_t{1} << lv) < groups) ++lv;
    p.levels = lv;
    p.units = static_cast<int>((v.T + p.tiles_per_unit - 1) / p.tiles_per_unit);
    if (o.mode == OUT_FULL && p.units != 1) return set_error(TBIK_BAD_ARGUMENT, "tc gemm: FULL needs 1 unit");
  }
  {  // raster knob (pure scheduling, same bits)
    const int64_t gm = knob(KNOB_TC_GROUP_M, GROUP_M);
    p.group_m = gm >= 1 ? static_cast<int>(gm) : GROUP_M;
  }
  const bool pair = tc_use_pair(v);
  p.tile_m = pair ? PAIR_M : BM;
  p.mblocks = static_cast<int>((v.M + p.tile_m - 1) / p.tile_m);
  p.ntiles = static_cast<int>((v.N + BN - 1) / BN);
  p.acc4 = p.levels == 0 && knob(KNOB_TC_ACC4, 1) != 0 ? 1 : 0;  // no level slot in TMEM: 4 accumulators
  p.items = static_cast<long long>(p.mblocks) * p.ntiles * p.units;
  const long long slots = pair ? sm_count() / 2 : sm_count();
  const long long nstreams = p.items < slots ? p.items : slots;
  dim3 grid(static_cast<unsigned>(pair ? 2 * nstreams : nstreams));
  const bool kf1 = p.kf == 1;
  // DEEP (see stages_for) when the items have at most 2 tree levels, or when there
  // are at most 2 waves of them: short launches are bound by load latency and the
  // extra stages pay for level 3 in scratch (K=14336, N=4096: M=256..1024 +5..9%,
  // M=2048 even; profiles/r01_tc_deep_midm.txt).  With 3+ levels and many waves
  // the on-chip level 3 measured faster (1146 vs 1108 TFLOP/s at the bench shape).
  // ... but not with 4+ levels (k_first = 1, K = 4096: 16 groups per item), where two
  // scratch levels cost more than the extra stages buy (tools/midm_sweep.py: o_proj
  // K=4096 N=4096 M=512..1024 +8-11 % without DEEP, down_proj K=14336 unchanged).
  // k_first == 1 keeps levels 1-3 off shared memory, so DEEP is free up to 3 levels
  // there and the shared-memory level 4 beats scratch above.  Knob tc_deep forces it.
  bool deep = kf1 ? p.levels <= 3 : p.levels <= 2 || (p.items <= 2 * slots && p.levels <= 3);
  {
    const int64_t k = knob(KNOB_TC_DEEP, -1);
    if (k == 0 || k == 1) deep = k == 1;
  }
  const int first_scratch = (kf1 ? 4 : 3) + (deep ? 0 : 1);
  if (p.levels >= first_scratch) {
    const size_t n = static_cast<size_t>(grid.x) * (p.levels - first_scratch + 1) * BM * BN;
    p.scratch = static_cast<float*>(workspace(n * sizeof(float), 1, s));
    if (!p.scratch) return set_error(TBIK_CUDA_ERROR, "tc gemm: scratch allocation failed");
  }
  // Results leave through a TMA store when the output is 16-byte addressable.
  CUtensorMap mC;
  std::memset(&mC, 0, sizeof(mC));
  const uint64_t ustride = o.mode != OUT_FULL ? static_cast<uint64_t>(o.unit_stride)
                                              : static_cast<uint64_t>(o.ldo) * static_cast<uint64_t>(v.M);
  p.tma_store = !o.act && (reinterpret_cast<uintptr_t>(o.out) & 15) == 0 && o.ldo % 4 == 0 && ustride % 4 == 0;
  if (p.tma_store)
    TBIK_TRY(make_map_out(&mC, o.out, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.M),
                          static_cast<uint64_t>(p.units), static_cast<uint64_t>(o.ldo) * 4, ustride * 4));
  int dev = 0;
  cudaGetDevice(&dev);
  using Kern = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcParams);
  // Fused GEMM -> tree all-reduce (tbik_group.cu) for FULL pair-tile launches whose
  // output is the group's send slot.
  if (FusedAr* ar = g_fused_ar) {
    bool ok = pair && abox == 128 && o.mode == OUT_FULL && !o.act && p.tma_store && o.ldo == v.N && ar->W > 1 &&
              ar->W <= 8 && p.items * 2 * ar->W <= ar->flag_capacity && o.out == ar->src[ar->rank];
    // Every CTA pair of every rank spins on peer tile flags before it exits, so the
    // whole grid must be co-resident: cap at the clusters the occupancy calculator
    // says fit (a static property of kernel and device, the same on every rank); a
    // grid that would not fit takes the separate path instead.
    if (ok) {
      static std::mutex mu;
      static std::map<int, int> max_clusters;
      std::lock_guard<std::mutex> lk(mu);
      auto f = max_clusters.find(dev);
      if (f == max_clusters.end()) {
        const Kern k = deep ? (kf1 ? tc_tree_gemm_kernel<true, 128, true, true, true>
                                   : tc_tree_gemm_kernel<false, 128, true, true, true>)
                            : (kf1 ? tc_tree_gemm_kernel<true, 128, true, false, true>
                                   : tc_tree_gemm_kernel<false, 128, true, false, true>);
        const size_t sm = smem_bytes(128, true, deep);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
        cudaLaunchConfig_t qc{};
        qc.gridDim = dim3(2);
        qc.blockDim = dim3(128 + 32 * EPI);
        qc.dynamicSmemBytes = sm;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = 2;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.attrs = qa;
        qc.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k, &qc) != cudaSuccess || n < 1) {
          cudaGetLastError();
          n = 1;
        }
        f = max_clusters.emplace(dev, n).first;
      }
      if (nstreams > f->second) ok = false;
    }
    if (ok) {
      p.ar_W = ar->W;
      p.ar_rank = ar->rank;
      p.ar_epoch = ar->epoch;
      for (int r = 0; r < 8; ++r) {
        p.ar_src[r] = ar->src[r];
        p.ar_dst[r] = ar->dst[r];
        p.ar_flags[r] = ar->flags[r];
        p.ar_done[r] = ar->done[r];
      }
      p.ar_counter = ar->counter;
      ar->used = true;
    }
  }
#define TBIK_TC_K(D, P)                                                                                        \
  {{tc_tree_gemm_kernel<false, 32, P, D>, tc_tree_gemm_kernel<true, 32, P, D>},                               \
   {tc_tree_gemm_kernel<false, 64, P, D>, tc_tree_gemm_kernel<true, 64, P, D>},                               \
   {tc_tree_gemm_kernel<false, 128, P, D>, tc_tree_gemm_kernel<true, 128, P, D>}}
  static const Kern table[2][2][3][2] = {{TBIK_TC_K(false, false), TBIK_TC_K(false, true)},
                                         {TBIK_TC_K(true, false), TBIK_TC_K(true, true)}};
#undef TBIK_TC_K
  const int ai = abox == 32 ? 0 : abox == 64 ? 1 : 2;
  const bool ar_on = p.ar_W > 1;
  const bool mse = p.ms_out != nullptr;
  if (mse && !(pair && abox == 128 && !ar_on))
    return set_error(TBIK_UNSUPPORTED, "tc gemm: the chunk (m, s) epilogue runs on 256-row pair tiles only");
  const Kern kern = mse ? (deep ? (kf1 ? tc_tree_gemm_kernel<true, 128, true, true, false, true>
                                       : tc_tree_gemm_kernel<false, 128, true, true, false, true>)
                                : (kf1 ? tc_tree_gemm_kernel<true, 128, true, false, false, true>
                                       : tc_tree_gemm_kernel<false, 128, true, false, false, true>))
                  : ar_on ? (deep ? (kf1 ? tc_tree_gemm_kernel<true, 128, true, true, true>
                                         : tc_tree_gemm_kernel<false, 128, true, true, true>)
                                  : (kf1 ? tc_tree_gemm_kernel<true, 128, true, false, true>
                                         : tc_tree_gemm_kernel<false, 128, true, false, true>))
                          : table[deep][pair][ai][kf1];
  const int nthreads = 128 + 32 * EPI;
  const size_t smem = smem_bytes(abox, pair, deep);
  if (!attr_done(dev, reinterpret_cast<const void*>(kern))) {
    TBIK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (pair) TBIK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = dim3(nthreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = !ar_on && knob(KNOB_TC_PDL, 1) != 0 ? 2 : 1;
  TBIK_CUDA(cudaLaunchKernelEx(&lc, kern, mA, mB, mC, p));
  count_launch(ar_on ? "tc_tree_gemm_kernel (fused all-reduce)" : "tc_tree_gemm_kernel");
  return TBIK_OK;
}

}  // namespace tbik_b200
