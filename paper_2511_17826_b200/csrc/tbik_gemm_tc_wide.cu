// tbik_gemm_tc_wide.cu -- the 256 x 256 pair-tile variant of the tcgen05 TBIK GEMM.
//
// Why a second kernel: the 256 x 128 kernel sits at ~14-15 TB/s of L2 -> SM
// crossbar traffic whether or not it merges (profiles/r01_tc_pipeline_ceiling.txt:
// 1221-1279 TFLOP/s with the merge switched off); a 256 x 256 pair tile pulls a
// third fewer bytes per flop (32 KB per 64-deep K step per SM for 2x the MMA work).
//
// TMEM (512 columns) holds ONE 128 x 256 f32 accumulator, split into two
// 128-column halves that the MMA issuer fills in turn (per K step: half 0's four
// N=128 MMAs, then half 1's), so half 0 of a leaf is drained by its four merge
// warps while half 1's last MMAs run, and half 1 while the next leaf's first
// half-0 MMAs run -- a single accumulator that never stalls the tensor pipe,
// leaving columns 256-511 for tree level 1.  Level 0 (the running leaf-group
// value) lives in the merge warps' registers, levels >= 2 (touched at most once
// per 2 groups) in L2-resident scratch; all of shared memory goes to operand
// stages.  When the last round of tiles would leave pairs idle, its tiles are
// split into 256 x 128 half items (one half of the accumulator / merge warps).
//
// Arithmetic is identical to the 256 x 128 kernel (tbik_gemm_tc.cu) -- the same
// tcgen05 N=128 K-step sequence per leaf half and the same __fadd_rn tree.
#include <mutex>
#include <string>

#include "tbik_common.cuh"
#include "tbik_internal.h"

namespace tbik_b200 {

namespace {

constexpr int BM = 128;
constexpr int PAIR_M = 256;
constexpr int BN = 256;
constexpr int KSTAGE = 64;
constexpr int KB_MAX = 4;  // K steps per accumulator-half block in the MMA issue order (p.kb <= 4)
constexpr int A_STAGE_BYTES = BM * KSTAGE * 2;  // 16 KB
constexpr int B_ATOM_BYTES = KSTAGE * 64 * 2;   // 8 KB
constexpr int B_STAGE_BYTES = 2 * B_ATOM_BYTES;  // 128 columns of B per CTA
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int EPI = 8;
constexpr int NUM_THREADS = 128 + 32 * EPI;
constexpr int COLS = 128;  // per merge thread
constexpr int TMEM_COLS = 512;
constexpr int GROUP_M = 8;
constexpr uint32_t IDESC = umma_idesc_bf16(PAIR_M, BN, /*a_mn_major=*/0, /*b_mn_major=*/1);
constexpr uint32_t IDESC_HALF = umma_idesc_bf16(PAIR_M, BN / 2, 0, 1);
constexpr size_t smem_bytes(int st) { return 1024 + static_cast<size_t>(st) * STAGE_BYTES + 256; }

struct WParams {
  int M, N, K;
  int bk, kf, T;
  int tiles_per_unit;
  int units;
  int mode;
  int levels;
  int mblocks, ntiles;
  long long items;
  long long full_items;  // items [0, full_items) are whole tiles, the rest halves
  long long split_base;  // whole-tile index of the first split tile
  float* out;
  long long ldo;
  long long unit_stride;
  float* scratch;  // [gridDim.x][levels - 1][BN/4][BM rows][4] (levels >= 2)
  int kb;          // K steps per half block (1, 2 or 4)
  int debug;       // TBIK_TC_DEBUG ablations: bit 0 skips the merge, bit 2 the tree above level 0
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* smem_dst, const CUtensorMap* map, uint32_t leader_bar,
                                                int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_2cta(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_2cta(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_2cta(uint32_t* smem_result, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc_2cta(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

struct Item {
  int m0, n0, unit, t_begin, t_end;
  int mask;  // active accumulator halves (bit h: columns n0 + 128h .. +128)
};

__device__ __forceinline__ Item decode(const WParams& p, long long item) {
  Item it;
  it.mask = 3;
  if (item >= p.full_items) {
    const long long j = item - p.full_items;
    it.mask = 1 << static_cast<int>(j & 1);
    item = p.split_base + (j >> 1);
  }
  it.unit = static_cast<int>(item % p.units);
  const long long rest = item / p.units;
  const long long group = GROUP_M * static_cast<long long>(p.ntiles);
  const int g = static_cast<int>(rest / group);
  const int idx = static_cast<int>(rest % group);
  const int gm = min(GROUP_M, p.mblocks - g * GROUP_M);
  const int mb = g * GROUP_M + idx % gm;
  const int nt = idx / gm;
  it.m0 = mb * PAIR_M;
  it.n0 = nt * BN;
  it.t_begin = it.unit * p.tiles_per_unit;
  it.t_end = min(p.T, it.t_begin + p.tiles_per_unit);
  return it;
}

__device__ __forceinline__ int tile_chunks(const WParams& p, int t) {
  const int kt0 = t * p.bk;
  const int kh = (kt0 + p.bk <= p.K) ? p.bk : p.K - kt0;
  return (kh + KSTAGE - 1) / KSTAGE;
}

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    tc_tree_gemm_wide_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const WParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // per accumulator half
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const long long pair = blockIdx.x >> 1;
  const long long npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&tfull[h], 1);
      mbar_init(&tempty[h], 2 * (EPI / 2));  // the half's merge warps in both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2cta(tmem_slot, TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      // per stage: A rows [am, am+128) x 64 K, and for each active half h the
      // 64 columns n0 + 128h + 64*rank (the pair's N=128 MMA B operand is split
      // across the two CTAs' shared memories)
      if (elect_one()) {
        const uint32_t full_leader0 = mapa(smem_u32(&full[0]), 0);
        int stage = 0;
        uint32_t phase = 0;
        for (long long item = pair; item < p.items; item += npairs) {
          const Item it = decode(p, item);
          const int am = it.m0 + static_cast<int>(rank) * BM;
          const uint32_t tx = A_STAGE_BYTES + (it.mask == 3 ? 2 : 1) * B_ATOM_BYTES;
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
              tma_load_2d_2sm(sA + stage * A_STAGE_BYTES, &tmA, fb, k, am);
#pragma unroll
              for (int h = 0; h < 2; ++h)
                if (it.mask >> h & 1)
                  tma_load_2d_2sm(sB + stage * B_STAGE_BYTES + h * B_ATOM_BYTES, &tmB, fb,
                                  it.n0 + h * 128 + static_cast<int>(rank) * 64, k);
              if (++stage == STAGES) {
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
      if (leader && elect_one()) {
        int stage = 0;
        uint32_t phase = 0;
        uint32_t hiter[2] = {0, 0};  // leaves accumulated so far per half
        for (long long item = pair; item < p.items; item += npairs) {
          const Item it = decode(p, item);
          for (int t = it.t_begin; t < it.t_end; ++t) {
            const int nch = tile_chunks(p, t);
            // K steps in blocks of KB: half 0's MMAs for the block, then half 1's.  A
            // half's last block ends 2*KB half-steps before the other half needs
            // the tensor pipe again, so each half is drained while the other half
            // computes (KB = 1 would leave the merge warps one N=128 K step).
            for (int c0 = 0; c0 < nch; c0 += p.kb) {
              const int nb = min(p.kb, nch - c0);
              int st[KB_MAX];
              uint32_t ph[KB_MAX];
#pragma unroll
              for (int j = 0; j < KB_MAX; ++j) {
                if (j >= nb) break;
                st[j] = stage;
                ph[j] = phase;
                if (++stage == STAGES) {
                  stage = 0;
                  phase ^= 1;
                }
              }
              int hdone = 0;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                if (!(it.mask >> h & 1)) continue;
                if (c0 == 0) {  // the half's previous leaf has been drained
                  mbar_wait(&tempty[h], (hiter[h] & 1) ^ 1);
                  tc_fence_after();
                }
#pragma unroll
                for (int j = 0; j < KB_MAX; ++j) {
                  if (j >= nb) break;
                  const int c = c0 + j;
                  if (hdone == 0) {  // first use of this stage
                    mbar_wait(&full[st[j]], ph[j]);
                    tc_fence_after();
                  }
                  const uint32_t a_base = smem_u32(sA + st[j] * A_STAGE_BYTES);
                  const uint32_t b_base = smem_u32(sB + st[j] * B_STAGE_BYTES) + h * B_ATOM_BYTES;
#pragma unroll
                  for (int kk = 0; kk < KSTAGE / 16; ++kk) {
                    const uint64_t adesc = umma_desc_sw128(a_base + kk * 32, 16, 1024);
                    const uint64_t bdesc = umma_desc_sw128(b_base + kk * 2048, B_ATOM_BYTES, 1024);
                    umma_bf16_2cta(tmem_base + h * 128, adesc, bdesc, IDESC_HALF, (c | kk) != 0 ? 1u : 0u);
                  }
                }
                if (c0 + nb == nch) {
                  umma_commit_2cta(&tfull[h], 0x3);
                  ++hiter[h];
                }
                ++hdone;
              }
#pragma unroll
              for (int j = 0; j < KB_MAX; ++j)
                if (j < nb) umma_commit_2cta(&empty[st[j]], 0x3);
            }
          }
        }
      }
      __syncwarp();
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    // ---------------- merge warps: 4 per accumulator half, one per TMEM lane quadrant ----------------
    const int ew = warp - 4;
    const int q = ew & 3;   // TMEM lanes 32q.. (a warp may only touch lanes 32*(warp%4)..)
    const int h = ew >> 2;  // accumulator half: columns 128h .. 128h + 127
    const int row_in_tile = q * 32 + lane;
    const int col0 = h * COLS;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t acc = lane_base + h * 128;
    const uint32_t slot1 = lane_base + 256 + h * 128;  // tree level 1
    const uint32_t tempty_leader = mapa(smem_u32(&tempty[h]), 0);
    // scratch slab per level >= 2: [col/4][row][4] -- a warp's float4 access is 512
    // contiguous bytes
    float* scratch_base = p.levels >= 2 ? p.scratch + static_cast<size_t>(blockIdx.x) * (p.levels - 1) * (BM * BN) +
                                              static_cast<size_t>(col0) * BM + static_cast<size_t>(row_in_tile) * 4
                                        : nullptr;
    float g[COLS];
    uint32_t hiter = 0;
    for (long long item = pair; item < p.items; item += npairs) {
      const Item it = decode(p, item);
      if (!(it.mask >> h & 1)) continue;
      const int grow = it.m0 + static_cast<int>(rank) * BM + row_in_tile;
      const bool row_ok = grow < p.M;
      const int ncols = min(COLS, p.N - it.n0 - col0);  // may be <= 0
      int t_in_group = 0;
      uint32_t groups_done = 0;
      for (int t = it.t_begin; t < it.t_end; ++t, ++hiter) {
        mbar_wait(&tfull[h], hiter & 1);
        tc_fence_after();
        if (p.mode == OUT_LEAVES) {
          float* dst = p.out + static_cast<size_t>(t) * p.unit_stride + static_cast<size_t>(grow) * p.ldo + it.n0 + col0;
#pragma unroll
          for (int c = 0; c < COLS / 32; ++c) {
            float v[32];
            tmem_ld32(acc + c * 32, v);
            if (row_ok) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c * 32 + i < ncols) dst[c * 32 + i] = v[i];
            }
          }
        } else if (!(p.debug & 1)) {
          // level 0: g = ((0 + P_0) + P_1) + ... (matmul.cpp:100-125), two 32-column
          // chunks in flight per wait
#pragma unroll
          for (int c = 0; c < COLS / 32; c += 2) {
            uint32_t r0[32], r1[32];
            tmem_ld32r(acc + c * 32, r0);
            tmem_ld32r(acc + c * 32 + 32, r1);
            tmem_wait_ld_dep(r0);
            tmem_wait_ld_dep(r1);
            if (t_in_group == 0) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                g[c * 32 + i] = __fadd_rn(0.0f, __uint_as_float(r0[i]));
                g[c * 32 + 32 + i] = __fadd_rn(0.0f, __uint_as_float(r1[i]));
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                g[c * 32 + i] = __fadd_rn(g[c * 32 + i], __uint_as_float(r0[i]));
                g[c * 32 + 32 + i] = __fadd_rn(g[c * 32 + 32 + i], __uint_as_float(r1[i]));
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader)
            mbar_arrive(&tempty[h]);
          else
            mbar_arrive_cluster(tempty_leader);
        }

        if (p.mode == OUT_LEAVES || (p.debug & 1)) continue;
        if (++t_in_group < p.kf) continue;
        t_in_group = 0;
        if (p.debug & 4) continue;  // ablation: level 0 only

        // Binary counter over completed groups (matmul.cpp:107-123): level 1 in
        // TMEM columns 256-511, deeper levels in scratch.
        int level = 1;
        uint32_t c_bits = groups_done++;
        while (c_bits & 1u) {
          if (level == 1) {
#pragma unroll
            for (int c = 0; c < COLS / 32; c += 2) {
              uint32_t r0[32], r1[32];
              tmem_ld32r(slot1 + c * 32, r0);
              tmem_ld32r(slot1 + c * 32 + 32, r1);
              tmem_wait_ld_dep(r0);
              tmem_wait_ld_dep(r1);
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                g[c * 32 + i] = __fadd_rn(g[c * 32 + i], __uint_as_float(r0[i]));
                g[c * 32 + 32 + i] = __fadd_rn(g[c * 32 + 32 + i], __uint_as_float(r1[i]));
              }
            }
          } else if (!(p.debug & 8)) {
            const float* sp = scratch_base + static_cast<size_t>(level - 2) * (BM * BN);
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
          if (level == 1) {
#pragma unroll
            for (int c = 0; c < COLS / 32; ++c) {
              float v[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = g[c * 32 + i];
              tmem_st32(slot1 + c * 32, v);
            }
            tmem_wait_st();
          } else if (!(p.debug & 16)) {
            float* sp = scratch_base + static_cast<size_t>(level - 2) * (BM * BN);
#pragma unroll
            for (int i = 0; i < COLS; i += 4)
              *reinterpret_cast<float4*>(sp + i * BM) = make_float4(g[i], g[i + 1], g[i + 2], g[i + 3]);
          }
          continue;
        }
        if (row_ok && ncols > 0 && !(p.debug & 32)) {
          float* dst = p.out + static_cast<size_t>(p.mode == OUT_UNITS ? it.unit : 0) * p.unit_stride +
                       static_cast<size_t>(grow) * p.ldo + it.n0 + col0;
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
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2cta(tmem_base, TMEM_COLS);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

tbik_status make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
                     uint32_t box_inner, uint32_t box_outer) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  if (!fn) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return TBIK_OK;
}

}  // namespace

int64_t tc_wide_pair_tiles(const GemmView& v) { return ((v.M + PAIR_M - 1) / PAIR_M) * ((v.N + BN - 1) / BN); }

tbik_status launch_tc_gemm_wide(const GemmView& v, const GemmOut& o, cudaStream_t s) {
  CUtensorMap mA, mB;
  TBIK_TRY(make_map(&mA, v.A, static_cast<uint64_t>(v.K), static_cast<uint64_t>(v.M), static_cast<uint64_t>(v.lda) * 2,
                    KSTAGE, BM));
  TBIK_TRY(make_map(&mB, v.B, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.K), static_cast<uint64_t>(v.ldb) * 2,
                    64, KSTAGE));
  WParams p{};
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
  p.mblocks = static_cast<int>((v.M + PAIR_M - 1) / PAIR_M);
  p.ntiles = static_cast<int>((v.N + BN - 1) / BN);
  const long long tiles = static_cast<long long>(p.mblocks) * p.ntiles * p.units;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long max_pairs = sms / 2;
  const long long npairs = tiles < max_pairs ? tiles : max_pairs;
  // Items go to pairs round-robin.  When the last round would leave at least half
  // of the pairs idle, its tiles become two half items each (TBIK_TC_WIDE_SPLIT=0
  // turns this off -- a pure scheduling knob).
  static const bool split_ok = [] {
    const char* e = std::getenv("TBIK_TC_WIDE_SPLIT");
    return !(e && *e == '0');
  }();
  const long long tail = tiles % npairs;
  if (split_ok && tiles > npairs && tail > 0 && 2 * tail <= npairs) {
    p.full_items = tiles - tail;
    p.split_base = tiles - tail;
    p.items = p.full_items + 2 * tail;
  } else {
    p.full_items = tiles;
    p.split_base = tiles;
    p.items = tiles;
  }
  dim3 grid(static_cast<unsigned>(2 * npairs));
  if (p.levels >= 2) {
    const size_t n = static_cast<size_t>(grid.x) * (p.levels - 1) * BM * BN;
    p.scratch = static_cast<float*>(workspace(n * sizeof(float), 1));
    if (!p.scratch) return set_error(TBIK_CUDA_ERROR, "tc gemm: scratch allocation failed");
  }
  static const int dbg = [] {
    const char* e = std::getenv("TBIK_TC_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  p.debug = dbg;
  static const int kb = [] {
    const char* e = std::getenv("TBIK_TC_WIDE_KB");
    const int v = e ? std::atoi(e) : 2;
    return v == 1 || v == 4 ? v : 2;
  }();
  p.kb = kb;
  // operand stages (TBIK_TC_WIDE_STAGES=4/5/6, a pure scheduling knob)
  static const int st = [] {
    const char* e = std::getenv("TBIK_TC_WIDE_STAGES");
    const int v = e ? std::atoi(e) : 6;
    return v == 4 || v == 5 ? v : 6;
  }();
  static bool attr_set[16][3] = {};
  if (dev >= 0 && dev < 16 && !attr_set[dev][st - 4]) {
    const void* fn = st == 4 ? reinterpret_cast<const void*>(tc_tree_gemm_wide_kernel<4>)
                   : st == 5 ? reinterpret_cast<const void*>(tc_tree_gemm_wide_kernel<5>)
                             : reinterpret_cast<const void*>(tc_tree_gemm_wide_kernel<6>);
    TBIK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes(st))));
    attr_set[dev][st - 4] = true;
  }
  if (st == 4)
    tc_tree_gemm_wide_kernel<4><<<grid, NUM_THREADS, smem_bytes(4), s>>>(mA, mB, p);
  else if (st == 5)
    tc_tree_gemm_wide_kernel<5><<<grid, NUM_THREADS, smem_bytes(5), s>>>(mA, mB, p);
  else
    tc_tree_gemm_wide_kernel<6><<<grid, NUM_THREADS, smem_bytes(6), s>>>(mA, mB, p);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

}  // namespace tbik_b200
