// tbik_gemm_tc_w.cu -- 256 x 256 pair tiles (N = 256 MMAs) for the tensor-core-leaf
// TBIK GEMM.
//
// Same arithmetic as tc_tree_gemm_kernel (tbik_gemm_tc.cu): every leaf is the
// block_k/16 tcgen05.mma.cta_group::2 K=16 steps into a zeroed TMEM accumulator,
// then the reference's fold and binary tree (matmul.cpp:100-125) in __fadd_rn.
// What changes is the MMA's N: 256 instead of 128.
//
// Why (profiles/r02_wide_tiles.md): the tensor core reads its shared-memory
// operands at ~64 B/clk per SM (ncu l1tex__data_pipe_tc_wavefronts_mem_shared: the
// 256 x 128 kernel and cuBLAS both sit at 0.5 wavefronts/clk).  An M=256 N=128 pair
// MMA needs A 4 KB + B 2 KB per SM per 64 clk = 96 B/clk, so that kernel's tensor
// pipe cannot exceed ~2/3 busy whatever the pipeline does -- exactly where it sat
// (67 %).  An N=256 MMA needs A 4 KB + B 4 KB per 128 clk = 64 B/clk: cuBLAS's
// operating point (97 % tensor-busy in the same capture).
//
// The price is TMEM: two 128 x 256 f32 accumulators per CTA fill all 512 columns,
// so the tree levels leave TMEM.  Level 1 (level 2 when k_first == 1, where level
// 1 is formed in registers) moves to shared memory -- 16 KB per merge warp, 128 KB
// per CTA -- which also serves as the output staging of the TMA stores once the
// tile's carry has consumed it; deeper levels (touched once per 4+ groups) live in
// L2-resident scratch.  That leaves 96 KB for operands: 3 stages of 64 K (A 16 KB +
// B 16 KB), 1536 MMA cycles in flight -- the same as the 256 x 128 kernel's 6
// stages of 256 cycles.
//
// Warp roles (384 threads, one CTA per SM, setmaxnreg 40 / 232):
//   warp 0      TMA producer (2SM TMA, completion on the leader's barrier)
//   warp 1      MMA issuer (leader CTA; whole warp loops, one lane issues)
//   warp 2      TMEM allocator
//   warps 4-11  merge warps: thread (w, lane) owns output row 32(w%4) + lane and the
//               128 columns [128 j, 128 j + 128), j = (w-4)/4, of the tile; g in 128
//               registers.
// Tail: when the last wave of 256 x 256 tiles would leave pairs idle, the remaining
// tiles run as 256 x 128 half items (N = 128 MMAs, merge warps j = 0 only) -- a
// schedule choice, the same bits (the MMA's N does not change any element's sum:
// tests/test_gpu_gemm.py::test_wide_tiles_bit_identical).
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "tbik_common.cuh"
#include "tbik_internal.h"
#include "tbik_pair.cuh"

namespace tbik_b200 {

tbik_status tc_make_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
tbik_status tc_make_map_out(CUtensorMap* map, float* base, uint64_t n, uint64_t m, uint64_t units,
                            uint64_t row_stride_bytes, uint64_t unit_stride_bytes);

namespace {

using namespace pair_ptx;

constexpr int BM = 128;     // rows per CTA (the pair covers 256)
constexpr int BNW = 256;    // columns per full tile (MMA N)
constexpr int HN = 128;     // columns per merge thread / per half item
constexpr int KSTAGE = 64;
constexpr int NST = 3;
constexpr int A_BYTES = BM * KSTAGE * 2;    // 16 KB
constexpr int BOX_BYTES = KSTAGE * 64 * 2;  // 8 KB: one 64-column B atom
constexpr int B_BYTES = 2 * BOX_BYTES;      // this CTA's 128 columns
constexpr int MERGE_WARPS = 8;
constexpr int NTHREADS = 128 + 32 * MERGE_WARPS;
constexpr int LVL_WARP_BYTES = 32 * HN * 4;  // 16 KB: one warp's 32 rows x 128 columns
constexpr int BOX_OUT = 32 * 32 * 4;         // 4 KB output staging box
constexpr int GROUP_M = 8;
constexpr uint32_t IDESC_FULL = umma_idesc_bf16(256, BNW, /*a_mn_major=*/0, /*b_mn_major=*/1);
constexpr uint32_t IDESC_HALF = umma_idesc_bf16(256, HN, 0, 1);
constexpr size_t SMEM_BYTES =
    1024 + static_cast<size_t>(NST) * (A_BYTES + B_BYTES) + static_cast<size_t>(MERGE_WARPS) * LVL_WARP_BYTES + 256;
static_assert(SMEM_BYTES <= 232448, "shared memory budget");

struct WParams {
  int M, N, K;
  int bk, kf, T;
  int tiles_per_unit;
  int units;
  int mode;    // OUT_FULL / OUT_UNITS
  int levels;  // log2(groups per unit)
  int mblocks, ntiles;  // 256-row blocks, 256-column tiles
  int group_m;
  long long full_items;  // items [0, full_items) are 256 x 256 tiles ...
  long long items;       // ... the rest 256 x 128 halves of the remaining tiles
  float* scratch;        // [gridDim.x][levels - FS + 1][BNW / 4][BM][4]
};

struct WItem {
  int m0, n0, unit, t_begin, t_end;
  bool wide;  // 256 columns, or a 128-column half item
};

__device__ __forceinline__ WItem decode(const WParams& p, long long item) {
  long long fi = item;
  int half = -1;
  if (item >= p.full_items) {
    const long long j = item - p.full_items;
    fi = p.full_items + j / 2;
    half = static_cast<int>(j & 1);
  }
  WItem it;
  it.unit = static_cast<int>(fi % p.units);
  const long long rest = fi / p.units;
  const long long group = static_cast<long long>(p.group_m) * p.ntiles;
  const int g = static_cast<int>(rest / group);
  const int idx = static_cast<int>(rest % group);
  const int gm = min(p.group_m, p.mblocks - g * p.group_m);
  it.m0 = (g * p.group_m + idx % gm) * 2 * BM;
  it.n0 = (idx / gm) * BNW + (half > 0 ? HN : 0);
  it.wide = half < 0;
  it.t_begin = it.unit * p.tiles_per_unit;
  it.t_end = min(p.T, it.t_begin + p.tiles_per_unit);
  return it;
}

__device__ __forceinline__ int tile_chunks(const WParams& p, int t) {
  const int kt0 = t * p.bk;
  const int kh = (kt0 + p.bk <= p.K) ? p.bk : p.K - kt0;
  return (kh + KSTAGE - 1) / KSTAGE;
}

__device__ __forceinline__ void ring_next(int& stage, uint32_t& phase) {
  if (++stage == NST) {
    stage = 0;
    phase ^= 1;
  }
}

template <bool KF1>
__global__ void __launch_bounds__(NTHREADS, 1)
    tc_wide_tree_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmC, const WParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + NST * A_BYTES;
  uint8_t* sLvl = sB + NST * B_BYTES;  // per merge warp: the shared-memory tree level / output staging
  uint64_t* full = reinterpret_cast<uint64_t*>(sLvl + MERGE_WARPS * LVL_WARP_BYTES);
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

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      if (elect_one()) {
        const uint32_t full_leader0 = mapa(smem_u32(&full[0]), leader_rank);
        int stage = 0;
        uint32_t phase = 0;
        for (long long item = pair; item < p.items; item += npairs) {
          const WItem it = decode(p, item);
          const int am = it.m0 + static_cast<int>(rank) * BM;
          // N = 256: CTA r stages columns [n0 + 128 r, +128) as two 64-column atoms;
          // N = 128 (half item): [n0 + 64 r, +64), one atom.
          const int bn = it.n0 + static_cast<int>(rank) * (it.wide ? HN : 64);
          const uint32_t tx = A_BYTES + (it.wide ? 2 : 1) * BOX_BYTES;
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
              tma_load_2d_2sm(sB + stage * B_BYTES, &tmB, fb, bn, k);
              if (it.wide) tma_load_2d_2sm(sB + stage * B_BYTES + BOX_BYTES, &tmB, fb, bn + 64, k);
              ring_next(stage, phase);
            }
          }
        }
      }
      __syncwarp();
    } else if (warp == 1 && leader) {
      // ---------------- MMA issuer (leader CTA) ----------------
      // Descriptors built once and advanced by constant offsets (see tbik_gemm_tc.cu).
      // B: MN-major SW128, 64-column atoms BOX_BYTES apart (LBO), 8-row K groups 1 KB
      // apart (SBO), +16 K rows (2 KB) per step.
      constexpr uint32_t DESC_HI = (1024u >> 4) | (1u << 14) | (2u << 29);
      const uint32_t a_lo0 = (smem_u32(sA) >> 4) | ((16u >> 4) << 16);
      const uint32_t b_lo0 = (smem_u32(sB) >> 4) | ((uint32_t(BOX_BYTES) >> 4) << 16);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc_iter = 0;
      for (long long item = pair; item < p.items; item += npairs) {
        const WItem it = decode(p, item);
        const uint32_t idesc = it.wide ? IDESC_FULL : IDESC_HALF;
        for (int t = it.t_begin; t < it.t_end; ++t, ++acc_iter) {
          const int buf = acc_iter & 1;
          mbar_wait(&tempty[buf], ((acc_iter >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + buf * BNW;
          const int nch = tile_chunks(p, t);
          for (int c = 0; c < nch; ++c) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a_lo = a_lo0 + static_cast<uint32_t>(stage) * (A_BYTES >> 4);
            const uint32_t b_lo = b_lo0 + static_cast<uint32_t>(stage) * (B_BYTES >> 4);
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < KSTAGE / 16; ++kk) {
                const uint64_t adesc = (static_cast<uint64_t>(DESC_HI) << 32) | (a_lo + kk * (32 >> 4));
                const uint64_t bdesc = (static_cast<uint64_t>(DESC_HI) << 32) | (b_lo + kk * (2048 >> 4));
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
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + j * HN;
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), leader_rank);
    constexpr int SL = KF1 ? 2 : 1;  // the shared-memory tree level
    constexpr int FS = SL + 1;       // first scratch level
    float* scratch_base =
        p.levels >= FS ? p.scratch +
                             static_cast<size_t>(blockIdx.x) * static_cast<size_t>(p.levels - FS + 1) * (BM * BNW) +
                             static_cast<size_t>(j * HN) * BM + static_cast<size_t>(row_in_tile) * 4
                       : nullptr;
    // [32 float4 columns][32 lanes][float4] (conflict-free 16-byte accesses); after
    // the tile's carry, four 128B-swizzled 32 x 32 output boxes
    uint8_t* lvl = sLvl + (warp - 4) * LVL_WARP_BYTES;
    float g[HN];
    uint32_t acc_iter = 0;
    for (long long item = pair; item < p.items; item += npairs) {
      const WItem it = decode(p, item);
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
        const uint32_t acc = lane_base + buf * BNW;
        const bool odd = KF1 && p.levels >= 1 && (groups_done & 1u);
        const bool first = KF1 || t_in_group == 0;
        // level 0: g = ((0 + P_0) + P_1) + ... + P_{kf-1}   (matmul.cpp:100-125); for
        // k_first == 1 an odd group merges with its even sibling kept in g (level 1
        // in registers): g = (0 + P) + g  (matmul.cpp:107-123, new + old)
#pragma unroll
        for (int cc = 0; cc < HN / 32; cc += 2) {
          uint32_t r[2][32];
          tmem_ld32r(acc + cc * 32, r[0]);
          tmem_ld32r(acc + cc * 32 + 32, r[1]);
          tmem_wait_ld_dep(r[0]);
          tmem_wait_ld_dep(r[1]);
          if (cc + 2 == HN / 32) {  // the accumulator is in registers: release it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (leader)
                mbar_arrive(&tempty[buf]);
              else
                mbar_arrive_cluster(tempty_leader0 + buf * 8);
            }
          }
          if (odd) {
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int i = 0; i < 32; ++i)
                g[(cc + u) * 32 + i] = __fadd_rn(__fadd_rn(0.0f, __uint_as_float(r[u][i])), g[(cc + u) * 32 + i]);
          } else if (first) {
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int i = 0; i < 32; ++i) g[(cc + u) * 32 + i] = __fadd_rn(0.0f, __uint_as_float(r[u][i]));
          } else {
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int i = 0; i < 32; ++i)
                g[(cc + u) * 32 + i] = __fadd_rn(g[(cc + u) * 32 + i], __uint_as_float(r[u][i]));
          }
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
            if (level == SL) {
#pragma unroll
              for (int i = 0; i < HN; i += 4) {
                const float4 x = *reinterpret_cast<const float4*>(lvl + ((i / 4) * 32 + lane) * 16);
                g[i] = __fadd_rn(g[i], x.x);
                g[i + 1] = __fadd_rn(g[i + 1], x.y);
                g[i + 2] = __fadd_rn(g[i + 2], x.z);
                g[i + 3] = __fadd_rn(g[i + 3], x.w);
              }
            } else {
              const float* sp = scratch_base + static_cast<size_t>(level - FS) * (BM * BNW);
#pragma unroll
              for (int i = 0; i < HN; i += 16) {
                float4 x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) x[u] = __ldcg(reinterpret_cast<const float4*>(sp + (i + 4 * u) * BM));
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  g[i + 4 * u] = __fadd_rn(g[i + 4 * u], x[u].x);
                  g[i + 4 * u + 1] = __fadd_rn(g[i + 4 * u + 1], x[u].y);
                  g[i + 4 * u + 2] = __fadd_rn(g[i + 4 * u + 2], x[u].z);
                  g[i + 4 * u + 3] = __fadd_rn(g[i + 4 * u + 3], x[u].w);
                }
              }
            }
            c_bits >>= 1;
            ++level;
          }
          if (level <= p.levels) {
            if (level == SL) {
              if (lane == 0) bulk_wait_read<0>();  // the previous tile's output boxes
              __syncwarp();
#pragma unroll
              for (int i = 0; i < HN; i += 4)
                *reinterpret_cast<float4*>(lvl + ((i / 4) * 32 + lane) * 16) =
                    make_float4(g[i], g[i + 1], g[i + 2], g[i + 3]);
            } else {
              float* sp = scratch_base + static_cast<size_t>(level - FS) * (BM * BNW);
#pragma unroll
              for (int i = 0; i < HN; i += 4)
                __stcg(reinterpret_cast<float4*>(sp + i * BM), make_float4(g[i], g[i + 1], g[i + 2], g[i + 3]));
            }
            continue;
          }
        }
        // The carry left the top level: g is this unit's complete (sub)tree.  The
        // shared-memory level is dead now; it stages four 32 x 32 boxes (128B swizzle,
        // conflict-free 16-byte stores) for TMA stores that clip ragged edges.
        __syncwarp();  // every lane's level reads are done
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int c = 0; c < HN / 32; ++c) {
          uint8_t* sbuf = lvl + c * BOX_OUT;
#pragma unroll
          for (int e = 0; e < 8; ++e)
            *reinterpret_cast<float4*>(sbuf + lane * 128 + ((e ^ (lane & 7)) << 4)) =
                make_float4(g[c * 32 + 4 * e], g[c * 32 + 4 * e + 1], g[c * 32 + 4 * e + 2], g[c * 32 + 4 * e + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int unit_out = p.mode == OUT_UNITS ? it.unit : 0;
#pragma unroll
          for (int c = 0; c < HN / 32; ++c)
            tma_store_3d(&tmC, smem_u32(lvl + c * BOX_OUT), col_base + c * 32, grow - lane, unit_out);
          bulk_commit();
        }
      }
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
// 256 x 232).  Checked once per (device, kernel); otherwise the wide path is off.
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
bool tc_wide_supported(const GemmView& v, const GemmOut& o) {
  const int64_t ustride = o.mode != OUT_FULL ? o.unit_stride : o.ldo * v.M;
  return (o.mode == OUT_FULL || o.mode == OUT_UNITS) && !o.act && !o.ms && v.M > BM &&
         (reinterpret_cast<uintptr_t>(o.out) & 15) == 0 && o.ldo % 4 == 0 && ustride % 4 == 0;
}

// Which pair-tile kernel a plain FULL / UNITS launch takes, and with how many K-split
// units (measured, profiles/r02_w192_tiles.md): 256 x 192 tiles whenever there are
// enough of them for the 74 CTA pairs -- >= 120 tiles (M=1024 N>=6144, M>=1536 N=4096:
// Llama down_proj M=4096 +10 %, M=1536 +15 %, lm_head M=1024 +8 %, TP shards +3..14 %,
// k_first = 1 shapes +4..12 %), or >= 80 tiles with K >= 8192 as two K units (M=1024:
// down_proj +2 %, Qwen3-32B down_proj K=25600 +48 %); otherwise the 256 x 128 kernel
// with its own split rule (M=1024 K=4096 N=4096: 41.5 vs 45.9 us).  256 x 256 tiles are
// never faster than 256 x 192 and remain a schedule option.  Knob tc_wide forces a
// variant (0 / 1 / 2), tc_units the split.
int64_t tc_w192_units(const GemmView& v) {
  if (v.M <= 128) return 0;
  const int64_t tiles = ((v.M + 255) / 256) * ((v.N + 191) / 192);
  if (tiles >= 120) return 1;
  if (tiles >= 80 && v.K >= 8192) return 2;
  return 0;
}

int tc_wide_variant(const GemmView& v) {
  const int64_t k = knob(KNOB_TC_WIDE, -1);
  if (k >= 0 && k <= 2) return static_cast<int>(k);
  return tc_w192_units(v) > 0 ? 2 : 0;
}

tbik_status launch_tc_wide(const GemmView& v, const GemmOut& o, cudaStream_t s) {
  if (!tc_wide_supported(v, o)) return set_error(TBIK_UNSUPPORTED, "tc wide: unsupported launch");
  const int kf1 = v.kf == 1;
  using Kern = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const WParams);
  const Kern kern = kf1 ? tc_wide_tree_gemm_kernel<true> : tc_wide_tree_gemm_kernel<false>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!regs_ok(dev, reinterpret_cast<const void*>(kern)))
    return set_error(TBIK_UNSUPPORTED, "tc wide: kernel register count is not 168");
  WParams p{};
  p.M = static_cast<int>(v.M);
  p.N = static_cast<int>(v.N);
  p.K = static_cast<int>(v.K);
  p.bk = static_cast<int>(v.bk);
  p.kf = static_cast<int>(v.kf);
  p.T = static_cast<int>(v.T);
  p.mode = o.mode;
  p.tiles_per_unit = static_cast<int>(o.tiles_per_unit);
  if (p.tiles_per_unit % p.kf) return set_error(TBIK_BAD_ARGUMENT, "tc wide: unit not whole groups");
  const int64_t groups = p.tiles_per_unit / p.kf;
  if (groups & (groups - 1)) return set_error(TBIK_BAD_ARGUMENT, "tc wide: unit not 2^j groups");
  int lv = 0;
  while ((int64_t{1} << lv) < groups) ++lv;
  p.levels = lv;
  p.units = static_cast<int>((v.T + p.tiles_per_unit - 1) / p.tiles_per_unit);
  if (o.mode == OUT_FULL && p.units != 1) return set_error(TBIK_BAD_ARGUMENT, "tc wide: FULL needs 1 unit");
  {
    const int64_t gm = knob(KNOB_TC_GROUP_M, GROUP_M);
    p.group_m = gm >= 1 ? static_cast<int>(gm) : GROUP_M;
  }
  p.mblocks = static_cast<int>((v.M + 2 * BM - 1) / (2 * BM));
  p.ntiles = static_cast<int>((v.N + BNW - 1) / BNW);
  const long long tiles = static_cast<long long>(p.mblocks) * p.ntiles * p.units;
  const long long slots = sm_count_dev() / 2;
  // Tail: split the last, partial wave into 256 x 128 halves when that shortens
  // the launch (waves counted in full-tile durations).
  p.full_items = tiles;
  {
    const long long r = tiles % slots;
    const double whole = static_cast<double>((tiles + slots - 1) / slots);
    const double split = static_cast<double>(tiles / slots) + 0.5 * static_cast<double>((2 * r + slots - 1) / slots);
    if (r > 0 && split < whole && knob(KNOB_TC_WIDE_TAIL, 1) != 0) p.full_items = tiles - r;
  }
  p.items = p.full_items + 2 * (tiles - p.full_items);
  const long long npairs = p.items < slots ? p.items : slots;
  const int FS = kf1 ? 3 : 2;
  if (p.levels >= FS) {
    const size_t n = static_cast<size_t>(2 * npairs) * (p.levels - FS + 1) * BM * BNW;
    p.scratch = static_cast<float*>(workspace(n * sizeof(float), 1, s));
    if (!p.scratch) return set_error(TBIK_CUDA_ERROR, "tc wide: scratch allocation failed");
  }
  CUtensorMap mA, mB, mC;
  TBIK_TRY(tc_make_map_2d(&mA, v.A, static_cast<uint64_t>(v.K), static_cast<uint64_t>(v.M),
                          static_cast<uint64_t>(v.lda) * 2, KSTAGE, BM));
  TBIK_TRY(tc_make_map_2d(&mB, v.B, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.K),
                          static_cast<uint64_t>(v.ldb) * 2, 64, KSTAGE));
  const uint64_t ustride = o.mode != OUT_FULL ? static_cast<uint64_t>(o.unit_stride)
                                              : static_cast<uint64_t>(o.ldo) * static_cast<uint64_t>(v.M);
  TBIK_TRY(tc_make_map_out(&mC, o.out, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.M),
                           static_cast<uint64_t>(p.units), static_cast<uint64_t>(o.ldo) * 4, ustride * 4));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(static_cast<unsigned>(2 * npairs));
  lc.blockDim = dim3(NTHREADS);
  lc.dynamicSmemBytes = SMEM_BYTES;
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  TBIK_CUDA(cudaLaunchKernelEx(&lc, kern, mA, mB, mC, p));
  count_launch("tc_wide_tree_gemm_kernel");
  return TBIK_OK;
}

}  // namespace tbik_b200
