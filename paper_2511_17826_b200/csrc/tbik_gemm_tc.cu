// tbik_gemm_tc.cu -- the TENSOR-CORE-LEAF TBIK GEMM for sm_100a.
//
// One CTA owns a 128 x 128 output tile and a K range (a "unit") of whole leaf
// tiles.  Warp roles (256 threads, one CTA per SM):
//   warp 0      TMA producer: A tile [128 m x 64 k] (K-major) and B tile
//               [64 k x 128 n] (the reference's row-major K x N weight, i.e.
//               MN-major for the MMA -- no pre-transpose) into a 6-stage
//               128B-swizzled shared-memory ring, completion on mbarriers.
//   warp 1      MMA issuer: for every leaf tile t, block_k/16 tcgen05.mma
//               (kind::f16, 128x128x16, bf16 -> f32) into a ZEROED TMEM
//               accumulator (first MMA with accumulate = 0).  Two accumulator
//               buffers (TMEM cols [0,128), [128,256)) so leaf t+1 is computed
//               while leaf t is merged.
//   warp 2      TMEM allocator (512 columns).
//   warps 4-7   merge warps: thread (q, lane) owns output row 32q + lane and
//               all 128 columns.  For every leaf they tcgen05.ld the leaf into
//               registers and apply the reference's reduction verbatim with
//               __fadd_rn:
//                 level 0   g = ((0 + P_0) + P_1) + ... + P_{kf-1}
//                           (TileReducer level 0, matmul.cpp:100-125)
//                 levels>=1 binary counter over group values, new + old
//                           (matmul.cpp:107-123; = T(.) of oracle.cpp:11-20)
//               g lives in 128 registers; pending tree levels 1 and 2 live in
//               TMEM (cols [256,384), [384,512)); deeper levels (touched once
//               per 8+ groups) spill to an L2-resident global scratch.
//
// Everything above the leaf is therefore bit-identical to the reference; the
// leaf P_t itself is the tensor core's block_k-long accumulation (DESIGN.md
// section 3 gives the measured ulp bound against leaf_dot).  Nothing in the
// per-element arithmetic depends on M, on the N position, on the unit split or
// on the TP shard, so the result is batch- and TP-invariant by construction.
#include <mutex>
#include <string>

#include "tbik_common.cuh"
#include "tbik_internal.h"

namespace tbik_b200 {

namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int KSTAGE = 64;  // K elements per pipeline stage (one 128 B swizzle row)
constexpr int STAGES = 6;
constexpr int A_STAGE_BYTES = BM * KSTAGE * 2;  // 16 KB
constexpr int B_STAGE_BYTES = KSTAGE * BN * 2;  // 16 KB (two 64-column boxes)
constexpr int B_BOX_BYTES = KSTAGE * 64 * 2;    // 8 KB
constexpr int NUM_THREADS = 256;
constexpr int TMEM_COLS = 512;
constexpr int SLOT_LVL1 = 256;
constexpr int SLOT_LVL2 = 384;
constexpr uint32_t IDESC = umma_idesc_bf16(BM, BN, /*a_mn_major=*/0, /*b_mn_major=*/1);
constexpr size_t SMEM_BYTES =
    1024 /*align slack*/ + STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 256 /*barriers*/;

struct TcParams {
  int M, N, K;
  int bk, kf, T;
  int tiles_per_unit;
  int mode;    // OUT_FULL / OUT_UNITS / OUT_LEAVES
  int levels;  // log2(groups per unit)
  float* out;
  long long ldo;
  long long unit_stride;
  float* scratch;  // [blocks][levels-2][BN][BM] when levels > 2
};

__device__ __forceinline__ int tile_chunks(const TcParams& p, int t) {
  const int kt0 = t * p.bk;
  const int kh = (kt0 + p.bk <= p.K) ? p.bk : p.K - kt0;
  return (kh + KSTAGE - 1) / KSTAGE;
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_tree_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN;
  const int m0 = blockIdx.y * BM;
  const int unit = blockIdx.z;
  const int t_begin = unit * p.tiles_per_unit;
  const int t_end = min(p.T, t_begin + p.tiles_per_unit);
  const int ntiles = t_end - t_begin;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_begin; t < t_end; ++t) {
        const int nch = tile_chunks(p, t);
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
          const int k = t * p.bk + c * KSTAGE;
          tma_load_2d(sA + stage * A_STAGE_BYTES, &tmA, &full[stage], k, m0);
          tma_load_2d(sB + stage * B_STAGE_BYTES, &tmB, &full[stage], n0, k);
          tma_load_2d(sB + stage * B_STAGE_BYTES + B_BOX_BYTES, &tmB, &full[stage], n0 + 64, k);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int lt = 0; lt < ntiles; ++lt) {
        const int buf = lt & 1;
        const uint32_t use = static_cast<uint32_t>(lt >> 1);
        mbar_wait(&tempty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * BN;
        const int nch = tile_chunks(p, t_begin + lt);
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_STAGE_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * B_STAGE_BYTES);
#pragma unroll
          for (int kk = 0; kk < KSTAGE / 16; ++kk) {
            // A: K-major SW128, +32 B per 16-element K step inside the atom.
            const uint64_t adesc = umma_desc_sw128(a_base + kk * 32, 16, 1024);
            // B: MN-major SW128, 64-column atoms 8 KB apart (LBO), 8-row K
            // groups 1 KB apart (SBO); +16 rows (2 KB) per K step.
            const uint64_t bdesc = umma_desc_sw128(b_base + kk * 2048, B_BOX_BYTES, 1024);
            umma_bf16(d, adesc, bdesc, IDESC, (c | kk) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------- merge warps (the TBIK reduction) ----------------
    const int q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    const int grow = m0 + row_in_tile;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const bool row_ok = grow < p.M;
    const int ncols = min(BN, p.N - n0);
    float g[BN];
#pragma unroll
    for (int i = 0; i < BN; ++i) g[i] = 0.0f;
    int t_in_group = 0;
    uint32_t groups_done = 0;
    float* scratch_base =
        p.levels > 2 ? p.scratch + (static_cast<size_t>(blockIdx.z) * gridDim.y * gridDim.x +
                                    static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) *
                                       static_cast<size_t>(p.levels - 2) * (BM * BN)
                     : nullptr;

    for (int lt = 0; lt < ntiles; ++lt) {
      const int buf = lt & 1;
      const uint32_t use = static_cast<uint32_t>(lt >> 1);
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const uint32_t acc = lane_base + buf * BN;
      if (p.mode == OUT_LEAVES) {
        float* dst = p.out + static_cast<size_t>(t_begin + lt) * p.unit_stride +
                     static_cast<size_t>(grow) * p.ldo + n0;
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          tmem_ld32(acc + c * 32, v);
          tmem_wait_ld();
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i < ncols) dst[c * 32 + i] = v[i];
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          tmem_ld32(acc + c * 32, v);
          tmem_wait_ld();
          if (t_in_group == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) g[c * 32 + i] = __fadd_rn(0.0f, v[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) g[c * 32 + i] = __fadd_rn(g[c * 32 + i], v[i]);
          }
        }
      }
      // Release the accumulator buffer to the MMA warp.
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);

      if (p.mode == OUT_LEAVES) continue;
      if (++t_in_group < p.kf) continue;
      t_in_group = 0;

      // Binary counter over completed groups (levels 1..p.levels).
      int level = 1;
      uint32_t c_bits = groups_done++;
      while (c_bits & 1u) {
        if (level <= 2) {
          const uint32_t slot = lane_base + (level == 1 ? SLOT_LVL1 : SLOT_LVL2);
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) {
            float v[32];
            tmem_ld32(slot + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) g[c * 32 + i] = __fadd_rn(g[c * 32 + i], v[i]);
          }
        } else {
          const float* s = scratch_base + static_cast<size_t>(level - 3) * (BM * BN) + row_in_tile;
#pragma unroll
          for (int i = 0; i < BN; ++i) g[i] = __fadd_rn(g[i], s[i * BM]);
        }
        c_bits >>= 1;
        ++level;
      }
      if (level <= p.levels) {
        if (level <= 2) {
          const uint32_t slot = lane_base + (level == 1 ? SLOT_LVL1 : SLOT_LVL2);
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = g[c * 32 + i];
            tmem_st32(slot + c * 32, v);
          }
          tmem_wait_st();
        } else {
          float* s = scratch_base + static_cast<size_t>(level - 3) * (BM * BN) + row_in_tile;
#pragma unroll
          for (int i = 0; i < BN; ++i) s[i * BM] = g[i];
        }
        continue;
      }
      // The carry left the top level: g is this unit's complete (sub)tree.
      if (row_ok) {
        float* dst = p.out + static_cast<size_t>(p.mode == OUT_UNITS ? unit : 0) * p.unit_stride +
                     static_cast<size_t>(grow) * p.ldo + n0;
        if (ncols == BN && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
          for (int i = 0; i < BN; i += 4)
            *reinterpret_cast<float4*>(dst + i) = make_float4(g[i], g[i + 1], g[i + 2], g[i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < BN; ++i)
            if (i < ncols) dst[i] = g[i];
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
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

tbik_status make_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                        uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TBIK_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return TBIK_OK;
}

}  // namespace

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

tbik_status launch_tc_gemm(const GemmView& v, const GemmOut& o, cudaStream_t s) {
  std::string why;
  if (!tc_supported(v, &why)) return set_error(TBIK_UNSUPPORTED, why);
  if (o.mode == OUT_GROUPS) return set_error(TBIK_BAD_ARGUMENT, "tc gemm: GROUPS mode is FMA-only");
  CUtensorMap mA, mB;
  TBIK_TRY(make_map_2d(&mA, v.A, static_cast<uint64_t>(v.K), static_cast<uint64_t>(v.M),
                       static_cast<uint64_t>(v.lda) * 2, KSTAGE, BM));
  TBIK_TRY(make_map_2d(&mB, v.B, static_cast<uint64_t>(v.N), static_cast<uint64_t>(v.K),
                       static_cast<uint64_t>(v.ldb) * 2, 64, KSTAGE));
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
  int64_t units;
  if (o.mode == OUT_LEAVES) {
    p.tiles_per_unit = 1;
    p.levels = 0;
    units = v.T;
  } else {
    p.tiles_per_unit = static_cast<int>(o.tiles_per_unit);
    if (p.tiles_per_unit % p.kf) return set_error(TBIK_BAD_ARGUMENT, "tc gemm: unit not whole groups");
    const int64_t groups = p.tiles_per_unit / p.kf;
    if (groups & (groups - 1)) return set_error(TBIK_BAD_ARGUMENT, "tc gemm: unit not 2^j groups");
    int lv = 0;
    while ((int64_t{1} << lv) < groups) ++lv;
    p.levels = lv;
    units = (v.T + p.tiles_per_unit - 1) / p.tiles_per_unit;
    if (o.mode == OUT_FULL && units != 1) return set_error(TBIK_BAD_ARGUMENT, "tc gemm: FULL needs 1 unit");
  }
  dim3 grid(static_cast<unsigned>((v.N + BN - 1) / BN), static_cast<unsigned>((v.M + BM - 1) / BM),
            static_cast<unsigned>(units));
  if (grid.y > 65535 || grid.z > 65535) return set_error(TBIK_UNSUPPORTED, "tc gemm: grid too large");
  if (p.levels > 2) {
    const size_t n = static_cast<size_t>(grid.x) * grid.y * grid.z * (p.levels - 2) * BM * BN;
    p.scratch = static_cast<float*>(workspace(n * sizeof(float), 1));
    if (!p.scratch) return set_error(TBIK_CUDA_ERROR, "tc gemm: scratch allocation failed");
  }
  static bool attr_set = false;
  if (!attr_set) {
    TBIK_CUDA(cudaFuncSetAttribute(tc_tree_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(SMEM_BYTES)));
    attr_set = true;
  }
  tc_tree_gemm_kernel<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(mA, mB, p);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

}  // namespace tbik_b200
