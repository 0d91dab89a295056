// tbik_gemm_tc_w192.cu -- 256 x 192 pair tiles (N = 192 MMAs) for the tensor-core-leaf
// TBIK GEMM.
//
// Same arithmetic as tc_tree_gemm_kernel (tbik_gemm_tc.cu): every leaf is the
// block_k/16 tcgen05.mma.cta_group::2 K=16 steps into a zeroed TMEM accumulator,
// then the reference's fold and binary tree (matmul.cpp:100-125) in __fadd_rn; the
// MMA's N changes no element's sum (tests/test_gpu_gemm.py: test_wide_tiles_bit_identical,
// test_wide_tiles_random_shapes, test_w192_tree_over_gpu_leaves).  Epilogues: f32
// output (FULL or K-split units) or the fused bf16 SiLU(gate)*up of interleaved
// gate/up columns.
//
// Why this width (profiles/r02_w192_tiles.md): the SM's shared-memory data port
// (~128 B/clk) carries the tensor core's operand reads AND the TMA writes of the same
// bytes.  Per CTA and 64-K stage a 256 x N pair tile moves A 16 KB + B N KB/8 twice,
// for 128 x N x 64 MACs:
//   N = 128 (tbik_gemm_tc.cu)   1.5 wavefronts per MMA cycle -> <= 67 % tensor-busy
//   N = 192 (this kernel)       1.17                         -> <= 85 %
//   N = 256                     1.0                          -> <= 100 %, but two
//                               accumulators fill TMEM and the tree levels then pay
//                               for shared memory through the same port (built and
//                               removed: profiles/r02_wide_tiles.md).
// At N = 192 two accumulators take 384 TMEM columns and the other 128 hold 2/3 of the
// tree level that is touched every other group (level 1; level 2 when k_first == 1);
// its last third (32 columns per thread) sits in shared memory -- a 4 KB slab per merge
// warp that also stages the output boxes of the TMA stores once the tile's carry has
// consumed the level.  The next level lives in 72 registers per thread + a 3 KB slab
// per warp (the accumulator is drained one 32-column chunk at a time to make room);
// deeper levels (touched once per 8+ groups) in L2-resident scratch.  Shared memory:
// 6 stages of {A 16 KB (128B swizzle), B 12 KB (three 32-column 64B-swizzle atoms; six
// 16-column 32B atoms for half items)} = 2304 MMA cycles in flight, 230.7 KB in all.
//
// Warp roles (384 threads, one CTA per SM, setmaxnreg 40 / 232):
//   warp 0      TMA producer (2SM TMA, completion on the leader's barrier)
//   warp 1      MMA issuer (leader CTA; whole warp loops, one lane issues)
//   warp 2      TMEM allocator
//   warps 4-11  merge warps: thread (w, lane) owns output row 32(w%4) + lane and the
//               96 columns [96 j, 96 j + 96), j = (w-4)/4, of the tile; g in 96 registers.
// Tail: when the last wave of tiles would leave pairs idle, the remaining tiles run as
// 256 x 96 half items (N = 96 MMAs, merge warps j = 0 only) -- a schedule choice.
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "tbik_common.cuh"
#include "tbik_internal.h"
#include "tbik_mathfn.cuh"
#include "tbik_pair.cuh"

namespace tbik_b200 {

tbik_status tc_make_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
tbik_status tc_make_map_2d_sw32(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                                uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
tbik_status tc_make_map_2d_sw64(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                                uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
tbik_status tc_make_map_out(CUtensorMap* map, float* base, uint64_t n, uint64_t m, uint64_t units,
                            uint64_t row_stride_bytes, uint64_t unit_stride_bytes);
tbik_status tc_make_map_act(CUtensorMap* map, uint16_t* base, uint64_t n, uint64_t m, uint64_t row_stride_bytes,
                            uint32_t box_n, uint32_t box_m);

namespace {

using namespace pair_ptx;

constexpr int BM = 128;      // rows per CTA (the pair covers 256)
constexpr int BNT = 192;     // columns per full tile (MMA N)
constexpr int HN = 96;       // columns per merge thread / per half item
constexpr int KSTAGE = 64;
constexpr int NST = 6;
constexpr int A_BYTES = BM * KSTAGE * 2;    // 16 KB
// B atoms: full tiles stage this CTA's 96 columns as three 32-column 64B-swizzle atoms
// (4 KB each), half items its 48 columns as three 16-column 32B-swizzle atoms (2 KB).
constexpr int ATOM_F = 32, ATOM_H = 16;
constexpr int ATOM_F_BYTES = ATOM_F * KSTAGE * 2;  // 4 KB
constexpr int ATOM_H_BYTES = ATOM_H * KSTAGE * 2;  // 2 KB
constexpr int B_BYTES = 3 * ATOM_F_BYTES;          // 12 KB: this CTA's 96 columns
constexpr int MERGE_WARPS = 8;
constexpr int NTHREADS = 128 + 32 * MERGE_WARPS;
constexpr int TCOLS = 64;                   // TMEM columns of the TMEM level per thread
constexpr int SCOLS = HN - TCOLS;           // shared-memory columns of it (32)
constexpr int LVL_WARP_BYTES = 32 * SCOLS * 4;  // 4 KB = one 32 x 32 f32 output box
constexpr int RCOLS = 72;                   // register columns of the register level per thread
constexpr int S2COLS = HN - RCOLS;          // its shared-memory columns (24)
constexpr int LVL2_WARP_BYTES = 32 * S2COLS * 4;  // 3 KB
constexpr int GROUP_M = 8;
constexpr uint32_t IDESC_FULL = umma_idesc_bf16(256, BNT, /*a_mn_major=*/0, /*b_mn_major=*/1);
constexpr uint32_t IDESC_HALF = umma_idesc_bf16(256, HN, 0, 1);
constexpr size_t SMEM_BYTES = 1024 + static_cast<size_t>(NST) * (A_BYTES + B_BYTES) +
                              static_cast<size_t>(MERGE_WARPS) * (LVL_WARP_BYTES + LVL2_WARP_BYTES) + 256;
static_assert(SMEM_BYTES <= 232448, "shared memory budget");
static_assert(2 * BNT + 2 * TCOLS == 512, "TMEM budget");

struct W3Params {
  int M, N, K;
  int bk, kf, T;
  int tiles_per_unit;
  int units;
  int mode;    // OUT_FULL / OUT_UNITS
  int levels;  // log2(groups per unit)
  int mblocks, ntiles;  // 256-row blocks, 192-column tiles
  int group_m;
  long long full_items;  // items [0, full_items) are 256 x 192 tiles ...
  long long items;       // ... the rest 256 x 96 halves of the remaining tiles
  float* scratch;        // [gridDim.x][levels - FS + 1][BNT / 4][BM][4]
  int act;               // 1: SiLU*up epilogue -- tmC maps the bf16 [M][N/2] output instead
};

struct W3Item {
  int m0, n0, unit, t_begin, t_end;
  bool wide;  // 192 columns, or a 96-column half item
};

__device__ __forceinline__ W3Item decode(const W3Params& p, long long item) {
  long long fi = item;
  int half = -1;
  if (item >= p.full_items) {
    const long long j = item - p.full_items;
    fi = p.full_items + j / 2;
    half = static_cast<int>(j & 1);
  }
  W3Item it;
  it.unit = static_cast<int>(fi % p.units);
  const long long rest = fi / p.units;
  const long long group = static_cast<long long>(p.group_m) * p.ntiles;
  const int g = static_cast<int>(rest / group);
  const int idx = static_cast<int>(rest % group);
  const int gm = min(p.group_m, p.mblocks - g * p.group_m);
  it.m0 = (g * p.group_m + idx % gm) * 2 * BM;
  it.n0 = (idx / gm) * BNT + (half > 0 ? HN : 0);
  it.wide = half < 0;
  it.t_begin = it.unit * p.tiles_per_unit;
  it.t_end = it.n0 < p.N ? min(p.T, it.t_begin + p.tiles_per_unit) : it.t_begin;  // a half past N: empty
  return it;
}

__device__ __forceinline__ int tile_chunks(const W3Params& p, int t) {
  const int kt0 = t * p.bk;
  const int kh = (kt0 + p.bk <= p.K) ? p.bk : p.K - kt0;
  return (kh + KSTAGE - 1) / KSTAGE;
}

// Scratch tree levels must survive in L2 while the streamed operands (one pass over A
// and W is about the L2's size) flow past them: stores carry an evict_last policy,
// the single read-back an evict_first one (the value is dead after it).
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_keep(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld_last(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol)
               : "memory");
  return v;
}

__device__ __forceinline__ void ring_next(int& stage, uint32_t& phase) {
  if (++stage == NST) {
    stage = 0;
    phase ^= 1;
  }
}

// One 32 x 32 f32 output box: registers -> 128B-swizzled staging (conflict-free
// 16-byte stores) -> TMA store (clips ragged edges).  The staging must be free: the
// caller waited for the previous store's read.
__device__ __forceinline__ void stage_and_store_box(uint8_t* stg, const float* v, const CUtensorMap* tmC, int col,
                                                    int row0, int unit, int lane) {
#pragma unroll
  for (int e = 0; e < 8; ++e)
    *reinterpret_cast<float4*>(stg + lane * 128 + ((e ^ (lane & 7)) << 4)) =
        make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(tmC, smem_u32(stg), col, row0, unit);
    bulk_commit();
  }
}

// Output box c (1 or 2) of the previous tile, parked in TMEM columns [32 (c-1), 32 c)
// of the thread's TMEM-level region, goes out through the staging.
__device__ __forceinline__ void emit_parked_box(uint8_t* stg, uint32_t lvl_t, int c, const CUtensorMap* tmC, int col,
                                                int row0, int unit, int lane) {
  uint32_t r[32];
  tmem_ld32r(lvl_t + (c - 1) * 32, r);
  tmem_wait_ld_dep(r);
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  __syncwarp();
  if (lane == 0) bulk_wait_read<0>();  // the previous box's read (long done: a leaf ago)
  __syncwarp();
  stage_and_store_box(stg, v, tmC, col + c * 32, row0, unit, lane);
}

template <bool KF1>
__global__ void __launch_bounds__(NTHREADS, 1)
    tc_w192_tree_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmC,
                             const W3Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + NST * A_BYTES;
  uint8_t* sLvl = sB + NST * B_BYTES;  // per merge warp: a third of the TMEM level / output staging
  uint8_t* sLvl2 = sLvl + MERGE_WARPS * LVL_WARP_BYTES;  // per merge warp: a quarter of the register level
  uint64_t* full = reinterpret_cast<uint64_t*>(sLvl2 + MERGE_WARPS * LVL2_WARP_BYTES);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1;
  const uint32_t leader_rank = crank & ~1u;
  const bool leader = rank == 0;
  const long long pair = blockIdx.x >> 1;
  const long long npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmBh);
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * MERGE_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2cta(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch (knob tc_pdl): the prologue above overlaps the
  // previous kernel's tail; operands, scratch and output are touched only after
  // it has completed.  Dependents may launch once every CTA got here (the grid is
  // co-resident), to run their own prologue on the SMs this grid frees.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      if (elect_one()) {
        const uint32_t full_leader0 = mapa(smem_u32(&full[0]), leader_rank);
        int stage = 0;
        uint32_t phase = 0;
        for (long long item = pair; item < p.items; item += npairs) {
          const W3Item it = decode(p, item);
          const int am = it.m0 + static_cast<int>(rank) * BM;
          // N = 192: CTA r stages columns [n0 + 96 r, +96) as three 32-column atoms;
          // N = 96 (half item): [n0 + 48 r, +48) as three 16-column atoms.
          const int atom = it.wide ? ATOM_F : ATOM_H;
          const int atom_bytes = it.wide ? ATOM_F_BYTES : ATOM_H_BYTES;
          const CUtensorMap* mb = it.wide ? &tmB : &tmBh;
          const int bn = it.n0 + static_cast<int>(rank) * 3 * atom;
          const uint32_t tx = A_BYTES + 3 * atom_bytes;
          for (int t = it.t_begin; t < it.t_end; ++t) {
            const int nch = tile_chunks(p, t);
            for (int c = 0; c < nch; ++c) {
              mbar_wait(&empty[stage], phase ^ 1);
              const uint32_t fb = full_leader0 + stage * 8;
              if (leader)
                mbar_arrive_expect_tx(&full[stage], tx);
              else
                mbar_arrive_expect_tx_cluster(fb, tx);
              const int k = t * p.bk + c * KSTAGE;
              tma_load_2d_2sm(sA + stage * A_BYTES, &tmA, fb, k, am);
              for (int a = 0; a < 3; ++a)
                tma_load_2d_2sm(sB + stage * B_BYTES + a * atom_bytes, mb, fb, bn + a * atom, k);
              ring_next(stage, phase);
            }
          }
        }
      }
      __syncwarp();
    } else if (warp == 1 && leader) {
      // ---------------- MMA issuer (leader CTA) ----------------
      // A: K-major SW128 (+32 B per K=16 step).  B: MN-major, atoms LBO apart, 8-row K
      // groups SBO apart: full tiles SW64 (LBO 4 KB, SBO 512 B, +1 KB per K=16 step),
      // half items SW32 (LBO 2 KB, SBO 256 B, +512 B).  Descriptors built once and
      // advanced by constant offsets.
      constexpr uint32_t A_HI = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t BF_HI = (512u >> 4) | (1u << 14) | (4u << 29);
      constexpr uint32_t BH_HI = (256u >> 4) | (1u << 14) | (6u << 29);
      const uint32_t a_lo0 = (smem_u32(sA) >> 4) | ((16u >> 4) << 16);
      const uint32_t bf_lo0 = (smem_u32(sB) >> 4) | ((uint32_t(ATOM_F_BYTES) >> 4) << 16);
      const uint32_t bh_lo0 = (smem_u32(sB) >> 4) | ((uint32_t(ATOM_H_BYTES) >> 4) << 16);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc_iter = 0;
      for (long long item = pair; item < p.items; item += npairs) {
        const W3Item it = decode(p, item);
        const uint32_t idesc = it.wide ? IDESC_FULL : IDESC_HALF;
        const uint32_t b_hi = it.wide ? BF_HI : BH_HI;
        const uint32_t b_lo0 = it.wide ? bf_lo0 : bh_lo0;
        const uint32_t b_step = it.wide ? (1024u >> 4) : (512u >> 4);
        for (int t = it.t_begin; t < it.t_end; ++t, ++acc_iter) {
          const int buf = acc_iter & 1;
          mbar_wait(&tempty[buf], ((acc_iter >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + buf * BNT;
          const int nch = tile_chunks(p, t);
          for (int c = 0; c < nch; ++c) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a_lo = a_lo0 + static_cast<uint32_t>(stage) * (A_BYTES >> 4);
            const uint32_t b_lo = b_lo0 + static_cast<uint32_t>(stage) * (B_BYTES >> 4);
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < KSTAGE / 16; ++kk) {
                const uint64_t adesc = (static_cast<uint64_t>(A_HI) << 32) | (a_lo + kk * (32 >> 4));
                const uint64_t bdesc = (static_cast<uint64_t>(b_hi) << 32) | (b_lo + kk * b_step);
                umma_bf16_2cta(d, adesc, bdesc, idesc, (c | kk) != 0 ? 1u : 0u);
              }
              umma_commit_2cta(&empty[stage], 0x3);
            }
            __syncwarp();
            ring_next(stage, phase);
          }
          if (elect_one()) umma_commit_2cta(&tfull[buf], static_cast<uint16_t>(0x3u << leader_rank));
          __syncwarp();
        }
      }
      __syncwarp();
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    // ---------------- merge warps (the TBIK reduction), both CTAs ----------------
    const int j = (warp - 4) >> 2;  // column half of the tile
    const int q = warp & 3;         // TMEM lane quarter 32*(warp%4)..
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t acc_base = tmem_base + lane_off + j * HN;
    const uint32_t lvl_t = tmem_base + lane_off + 2 * BNT + j * TCOLS;  // TMEM part of the TMEM level
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), leader_rank);
    constexpr int TL = KF1 ? 2 : 1;  // the TMEM (+ shared-memory third) tree level
    constexpr int RLV = TL + 1;      // the register (+ shared-memory quarter) level
    constexpr int FS = TL + 2;       // first scratch level
    float* scratch_base =
        p.levels >= FS ? p.scratch +
                             static_cast<size_t>(blockIdx.x) * static_cast<size_t>(p.levels - FS + 1) * (BM * BNT) +
                             static_cast<size_t>(j * HN) * BM + static_cast<size_t>(row_in_tile) * 4
                       : nullptr;
    // shared-memory third of the TMEM level: [8 float4 columns][32 lanes][float4]; after
    // the tile's carry, one 128B-swizzled 32 x 32 output box
    uint8_t* lvl_s = sLvl + (warp - 4) * LVL_WARP_BYTES;
    uint8_t* lvl2_s = sLvl2 + (warp - 4) * LVL2_WARP_BYTES;
    float l2r[RCOLS];
    const uint64_t pol_last = l2_policy_evict_last();
    const uint64_t pol_first = l2_policy_evict_first();
    float g[HN];
    uint32_t acc_iter = 0;
    // Output boxes 1-2 of the last finished tile wait in the (then dead) TMEM-level
    // columns and leave one per following leaf: the staging then never waits for a
    // TMA read in flight (three back-to-back boxes through one 4 KB staging cost the
    // tile's end ~3 store round trips).  The TMEM level is first rewritten no earlier
    // than the second leaf of the next tile, after both have left.
    int parked = 0, pk_col = 0, pk_row = 0, pk_unit = 0;
    for (long long item = pair; item < p.items; item += npairs) {
      const W3Item it = decode(p, item);
      const bool mine = it.wide || j == 0;
      const int col_base = it.n0 + (it.wide ? j * HN : 0);
      const int grow = it.m0 + static_cast<int>(rank) * BM + row_in_tile;
      int t_in_group = 0;
      uint32_t groups_done = 0;
      for (int t = it.t_begin; t < it.t_end; ++t, ++acc_iter) {
        const int buf = acc_iter & 1;
        mbar_wait(&tfull[buf], (acc_iter >> 1) & 1);
        tc_fence_after();
        if (!mine) {  // a half item: the other half's warps only hand the slot back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader)
              mbar_arrive(&tempty[buf]);
            else
              mbar_arrive_cluster(tempty_leader0 + buf * 8);
          }
          continue;
        }
        const uint32_t acc = acc_base + buf * BNT;
        const bool odd = KF1 && p.levels >= 1 && (groups_done & 1u);
        const bool first = KF1 || t_in_group == 0;
        {
          // one 32-column chunk at a time (the register level needs the room), each
          // folded as it arrives; the accumulator goes back after the last load
          uint32_t r[HN / 32][32];
#pragma unroll
          for (int c = 0; c < HN / 32; ++c) {
            tmem_ld32r(acc + c * 32, r[c]);
            tmem_wait_ld_dep(r[c]);
            if (c == HN / 32 - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                if (leader)
                  mbar_arrive(&tempty[buf]);
                else
                  mbar_arrive_cluster(tempty_leader0 + buf * 8);
              }
            }
            // level 0: g = ((0 + P_0) + P_1) + ... + P_{kf-1}   (matmul.cpp:100-125); for
            // k_first == 1 an odd group merges with its even sibling kept in g (level 1
            // in registers): g = (0 + P) + g  (matmul.cpp:107-123, new + old)
            if (odd) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                g[c * 32 + i] = __fadd_rn(__fadd_rn(0.0f, __uint_as_float(r[c][i])), g[c * 32 + i]);
            } else if (first) {
#pragma unroll
              for (int i = 0; i < 32; ++i) g[c * 32 + i] = __fadd_rn(0.0f, __uint_as_float(r[c][i]));
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) g[c * 32 + i] = __fadd_rn(g[c * 32 + i], __uint_as_float(r[c][i]));
            }
          }
        }
        if (parked > 0) {  // next parked box of the previous tile (3 - parked = 1, then 2)
          emit_parked_box(lvl_s, lvl_t, 3 - parked, &tmC, pk_col, pk_row, pk_unit, lane);
          --parked;
        }
        if (!KF1 && ++t_in_group < p.kf) continue;
        t_in_group = 0;
        // Binary counter over completed groups (levels 1..p.levels, matmul.cpp:107-123).
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
            if (level == TL) {
              uint32_t r[TCOLS / 32][32];
#pragma unroll
              for (int c = 0; c < TCOLS / 32; ++c) tmem_ld32r(lvl_t + c * 32, r[c]);
#pragma unroll
              for (int c = 0; c < TCOLS / 32; ++c) tmem_wait_ld_dep(r[c]);
#pragma unroll
              for (int c = 0; c < TCOLS / 32; ++c)
#pragma unroll
                for (int i = 0; i < 32; ++i) g[c * 32 + i] = __fadd_rn(g[c * 32 + i], __uint_as_float(r[c][i]));
#pragma unroll
              for (int i = 0; i < SCOLS; i += 4) {
                const float4 x = *reinterpret_cast<const float4*>(lvl_s + ((i / 4) * 32 + lane) * 16);
                g[TCOLS + i] = __fadd_rn(g[TCOLS + i], x.x);
                g[TCOLS + i + 1] = __fadd_rn(g[TCOLS + i + 1], x.y);
                g[TCOLS + i + 2] = __fadd_rn(g[TCOLS + i + 2], x.z);
                g[TCOLS + i + 3] = __fadd_rn(g[TCOLS + i + 3], x.w);
              }
            } else if (level == RLV) {
#pragma unroll
              for (int i = 0; i < RCOLS; ++i) g[i] = __fadd_rn(g[i], l2r[i]);
#pragma unroll
              for (int i = 0; i < S2COLS; i += 4) {
                const float4 x = *reinterpret_cast<const float4*>(lvl2_s + ((i / 4) * 32 + lane) * 16);
                g[RCOLS + i] = __fadd_rn(g[RCOLS + i], x.x);
                g[RCOLS + i + 1] = __fadd_rn(g[RCOLS + i + 1], x.y);
                g[RCOLS + i + 2] = __fadd_rn(g[RCOLS + i + 2], x.z);
                g[RCOLS + i + 3] = __fadd_rn(g[RCOLS + i + 3], x.w);
              }
            } else {
              // all 24 loads in flight at once: one L2 round trip per level, not six
              const float* sp = scratch_base + static_cast<size_t>(level - FS) * (BM * BNT);
              constexpr int NB = 2;  // two batches of loads (register room)
#pragma unroll
              for (int b = 0; b < NB; ++b) {
                float4 x[HN / 4 / NB];
#pragma unroll
                for (int u = 0; u < HN / 4 / NB; ++u) x[u] = ld_last(sp + 4 * (b * HN / 4 / NB + u) * BM, pol_first);
#pragma unroll
                for (int u = 0; u < HN / 4 / NB; ++u) {
                  const int c = 4 * (b * HN / 4 / NB + u);
                  g[c] = __fadd_rn(g[c], x[u].x);
                  g[c + 1] = __fadd_rn(g[c + 1], x[u].y);
                  g[c + 2] = __fadd_rn(g[c + 2], x[u].z);
                  g[c + 3] = __fadd_rn(g[c + 3], x[u].w);
                }
              }
            }
            c_bits >>= 1;
            ++level;
          }
          if (level <= p.levels) {
            if (level == TL) {
#pragma unroll
              for (int c = 0; c < TCOLS / 32; ++c) {
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = g[c * 32 + i];
                tmem_st32(lvl_t + c * 32, v);
              }
              if (lane == 0) bulk_wait_read<0>();  // the previous tile's output box
              __syncwarp();
#pragma unroll
              for (int i = 0; i < SCOLS; i += 4)
                *reinterpret_cast<float4*>(lvl_s + ((i / 4) * 32 + lane) * 16) =
                    make_float4(g[TCOLS + i], g[TCOLS + i + 1], g[TCOLS + i + 2], g[TCOLS + i + 3]);
              tmem_wait_st();
            } else if (level == RLV) {
#pragma unroll
              for (int i = 0; i < RCOLS; ++i) l2r[i] = g[i];
#pragma unroll
              for (int i = 0; i < S2COLS; i += 4)
                *reinterpret_cast<float4*>(lvl2_s + ((i / 4) * 32 + lane) * 16) =
                    make_float4(g[RCOLS + i], g[RCOLS + i + 1], g[RCOLS + i + 2], g[RCOLS + i + 3]);
            } else {
              float* sp = scratch_base + static_cast<size_t>(level - FS) * (BM * BNT);
#pragma unroll
              for (int i = 0; i < HN; i += 4)
                st_keep(sp + i * BM, make_float4(g[i], g[i + 1], g[i + 2], g[i + 3]), pol_last);
            }
            continue;
          }
        }
        // The carry left the top level: g is this unit's complete (sub)tree.  The
        // shared-memory third of the level is dead now; it stages the three 32 x 32
        // output boxes one after the other (128B swizzle, conflict-free 16-byte stores)
        // for TMA stores that clip ragged edges.
        const int unit_out = p.mode == OUT_UNITS ? it.unit : 0;
        if (p.act) {
          // fused SiLU(gate) * up (tb_silu_mul_bf16, the same ops as tbik_silu_mul): the
          // thread's 96 columns are 48 (gate, up) pairs -> 48 bf16 = one 96-byte row of a
          // 32 x 48 bf16 box staged in the dead level slab, one TMA store per warp
          __syncwarp();
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
#pragma unroll
          for (int q8 = 0; q8 < HN / 16; ++q8) {
            uint32_t w4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = q8 * 16 + 4 * e;
              w4[e] = static_cast<uint32_t>(tb_silu_mul_bf16(g[c], g[c + 1])) |
                      (static_cast<uint32_t>(tb_silu_mul_bf16(g[c + 2], g[c + 3])) << 16);
            }
            *reinterpret_cast<uint4*>(lvl_s + lane * (HN / 2 * 2) + q8 * 16) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmC, smem_u32(lvl_s), col_base / 2, grow - lane, 0);
            bulk_commit();
          }
          continue;
        }
        while (parked > 0) {  // a tile of a single leaf: the previous tile's boxes go first
          emit_parked_box(lvl_s, lvl_t, 3 - parked, &tmC, pk_col, pk_row, pk_unit, lane);
          --parked;
        }
        // box 0 now; boxes 1-2 parked in the dead TMEM-level columns
#pragma unroll
        for (int c = 1; c < HN / 32; ++c) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = g[c * 32 + i];
          tmem_st32(lvl_t + (c - 1) * 32, v);
        }
        __syncwarp();  // every lane's reads of the staging region are done
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
        stage_and_store_box(lvl_s, g, &tmC, col_base, grow - lane, unit_out, lane);
        tmem_wait_st();
        parked = HN / 32 - 1;
        pk_col = col_base;
        pk_row = grow - lane;
        pk_unit = unit_out;
      }
    }
    while (parked > 0) {
      emit_parked_box(lvl_s, lvl_t, 3 - parked, &tmC, pk_col, pk_row, pk_unit, lane);
      --parked;
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2cta(tmem_base, 512);
  }
}

int sm_count_dev() {
  static int n[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  if (dev >= 0 && dev < 16) {
    if (!n[dev]) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
    if (n[dev]) sms = n[dev];
  }
  return sms;
}

// setmaxnreg only redistributes the registers the launch allocated: the merge
// warpgroups' 232 need exactly 168 per thread at launch (384 x 168 = 128 x 40 +
// 256 x 232).  Checked once per (device, kernel); otherwise this path is off.
bool regs_ok(int dev, const void* kern) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> ok;
  std::lock_guard<std::mutex> lk(mu);
  auto f = ok.find({dev, kern});
  if (f != ok.end()) return f->second;
  cudaFuncAttributes fa{};
  const bool good = cudaFuncGetAttributes(&fa, kern) == cudaSuccess && fa.numRegs == 168;
  if (!good) cudaGetLastError();
  ok[{dev, kern}] = good;
  if (good) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SMEM_BYTES));
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
  }
  return good;
}

}  // namespace

// FULL / UNITS launches of pair tiles with a 16-byte addressable f32 output (TMA
// stores) and no epilogue; any block_k (the stage ring streams a leaf).
// The lm_head's chunk (m, s) epilogue stays on the 256x128 kernel: on 256x192 tiles
// its exp work at the tile end cost more than the tile saves (M=1024 K=4096 V=128256:
// 1083.6 vs 1062.5 us, tools/lm_head_w192.py).
bool tc_wide_supported(const GemmView& v, const GemmOut& o) {
  if (o.ms || v.M <= BM) return false;
  if (o.act)  // the SiLU*up epilogue: FULL, even N, a 16-byte addressable bf16 output
    return o.mode == OUT_FULL && v.N % 2 == 0 && (reinterpret_cast<uintptr_t>(o.act) & 15) == 0 && o.ld_act % 8 == 0;
  const int64_t ustride = o.mode != OUT_FULL ? o.unit_stride : o.ldo * v.M;
  return (o.mode == OUT_FULL || o.mode == OUT_UNITS) && (reinterpret_cast<uintptr_t>(o.out) & 15) == 0 &&
         o.ldo % 4 == 0 && ustride % 4 == 0;
}

// Which pair-tile kernel a plain FULL / UNITS launch takes, and with how many K-split
// units (measured, profiles/r02_w192_tiles.md): 256 x 192 tiles whenever there are
// enough of them for the 74 CTA pairs -- >= 120 tiles (M=1024 N>=6144, M>=1536 N=4096:
// Llama down_proj M=4096 +10 %, M=1536 +15 %, lm_head M=1024 +8 %, TP shards +3..14 %,
// k_first = 1 shapes +4..12 %), or >= 80 tiles with K >= 8192 as two K units (M=1024:
// down_proj +2 %, Qwen3-32B down_proj K=25600 +48 %); otherwise the 256 x 128 kernel
// with its own split rule (M=1024 K=4096 N=4096: 41.5 vs 45.9 us).  256 x 256 tiles are
// never faster than 256 x 192 (built, measured and removed in round 2:
// profiles/r02_wide_tiles.md).  Knob tc_wide forces the choice (0: 256 x 128,
// 1: 256 x 192), tc_units the split.
int64_t tc_w192_units(const GemmView& v) {
  if (v.M <= 128) return 0;
  const int64_t tiles = ((v.M + 255) / 256) * ((v.N + 191) / 192);
  if (tiles >= 120) return 1;
  if (tiles >= 80 && v.K >= 8192) return 2;
  return 0;
}

int tc_wide_variant(const GemmView& v) {
  const int64_t k = knob(KNOB_TC_WIDE, -1);
  if (k == 0) return 0;
  if (k >= 1) return 1;
  return tc_w192_units(v) > 0 ? 1 : 0;
}

tbik_status launch_tc_w192(const GemmView& v, const GemmOut& o, cudaStream_t s) {
  if (!tc_wide_supported(v, o)) return set_error(TBIK_UNSUPPORTED, "tc w192: unsupported launch");
  const int kf1 = v.kf == 1;
  using Kern = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap, const W3Params);
  const Kern kern = kf1 ? tc_w192_tree_gemm_kernel<true> : tc_w192_tree_gemm_kernel<false>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!regs_ok(dev, reinterpret_cast<const void*>(kern)))
    return set_error(TBIK_UNSUPPORTED, "tc w192: kernel register count is not 168");
  W3Params p{};
  p.M = static_cast<int>(v.M);
  p.N = static_cast<int>(v.N);
  p.K = static_cast<int>(v.K);
  p.bk = static_cast<int>(v.bk);
  p.kf = static_cast<int>(v.kf);
  p.T = static_cast<int>(v.T);
  p.mode = o.mode;
  p.tiles_per_unit = static_cast<int>(o.tiles_per_unit);
  if (p.tiles_per_unit % p.kf) return set_error(TBIK_BAD_ARGUMENT, "tc w192: unit not whole groups");
  const int64_t groups = p.tiles_per_unit / p.kf;
  if (groups & (groups - 1)) return set_error(TBIK_BAD_ARGUMENT, "tc w192: unit not 2^j groups");
  int lv = 0;
  while ((int64_t{1} << lv) < groups) ++lv;
  p.levels = lv;
  p.units = static_cast<int>((v.T + p.tiles_per_unit - 1) / p.tiles_per_unit);
  if (o.mode == OUT_FULL && p.units != 1) return set_error(TBIK_BAD_ARGUMENT, "tc w192: FULL needs 1 unit");
  {
    const int64_t gm = knob(KNOB_TC_GROUP_M, GROUP_M);
    p.group_m = gm >= 1 ? static_cast<int>(gm) : GROUP_M;
  }
  p.mblocks = static_cast<int>((v.M + 2 * BM - 1) / (2 * BM));
  p.ntiles = static_cast<int>((v.N + BNT - 1) / BNT);
  const long long tiles = static_cast<long long>(p.mblocks) * p.ntiles * p.units;
  const long long slots = sm_count_dev() / 2;
  // Tail: split the last, partial wave into 256 x 96 halves when that shortens the
  // launch (waves counted in full-tile durations).
  p.full_items = tiles;
  {
    const long long r = tiles % slots;
    const double whole = static_cast<double>((tiles + slots - 1) / slots);
    const double split = static_cast<double>(tiles / slots) + 0.5 * static_cast<double>((2 * r + slots - 1) / slots);
    if (r > 0 && split < whole && knob(KNOB_TC_WIDE_TAIL, 1) != 0) p.full_items = tiles - r;
  }
  p.items = p.full_items + 2 * (tiles - p.full_items);
  const long long npairs = p.items < slots ? p.items : slots;
  const int FS = kf1 ? 4 : 3;
  if (p.levels >= FS) {
    const size_t n = static_cast<size_t>(2 * npairs) * (p.levels - FS + 1) * BM * BNT;
    p.scratch = static_cast<float*>(workspace(n * sizeof(float), 1, s));
    if (!p.scratch) return set_error(TBIK_CUDA_ERROR, "tc w192: scratch allocation failed");
  }
  CUtensorMap mA, mB, mBh, mC;
  TBIK_TRY(tc_make_map_2d(&mA, v.A, static_cast<uint64_t>(v.K), static_cast<uint64_t>(v.M),
                          static_cast<uint64_t>(v.lda) * 2, KSTAGE, BM));
  TBIK_TRY(tc_make_map_2d_sw64(&mB, v.B, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.K),
                               static_cast<uint64_t>(v.ldb) * 2, ATOM_F, KSTAGE));
  TBIK_TRY(tc_make_map_2d_sw32(&mBh, v.B, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.K),
                               static_cast<uint64_t>(v.ldb) * 2, ATOM_H, KSTAGE));
  if (o.act) {
    p.act = 1;
    TBIK_TRY(tc_make_map_act(&mC, o.act, static_cast<uint64_t>(v.N / 2), static_cast<uint64_t>(v.M),
                             static_cast<uint64_t>(o.ld_act) * 2, HN / 2, 32));
  } else {
    const uint64_t ustride = o.mode != OUT_FULL ? static_cast<uint64_t>(o.unit_stride)
                                                : static_cast<uint64_t>(o.ldo) * static_cast<uint64_t>(v.M);
    TBIK_TRY(tc_make_map_out(&mC, o.out, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.M),
                             static_cast<uint64_t>(p.units), static_cast<uint64_t>(o.ldo) * 4, ustride * 4));
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(static_cast<unsigned>(2 * npairs));
  lc.blockDim = dim3(NTHREADS);
  lc.dynamicSmemBytes = SMEM_BYTES;
  lc.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = knob(KNOB_TC_PDL, 1) != 0 ? 2 : 1;
  TBIK_CUDA(cudaLaunchKernelEx(&lc, kern, mA, mB, mBh, mC, p));
  count_launch("tc_w192_tree_gemm_kernel");
  return TBIK_OK;
}

}  // namespace tbik_b200
