// tbik_internal.h -- launcher interfaces shared by the C ABI translation unit
// and the kernel translation units.  Not installed; not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "tbik_b200.h"

namespace tbik_b200 {

constexpr int kMaxRanks = 64;

struct PartPtrs {
  const float* p[kMaxRanks];
};

// Output layout of one GEMM launch.  A "unit" is the K range one CTA column
// reduces:
//   OUT_FULL    all tiles of the view, full tree  -> C[M x N] (ldo)
//   OUT_UNITS   2^j whole leaf groups per unit    -> subtree value -> ws[unit][M][N]
//   OUT_LEAVES  one tile per unit                 -> P_t          -> ws[t][M][N]
//   OUT_GROUPS  one leaf group per unit (FMA)     -> group value  -> ws[g][M][N]
enum OutMode { OUT_FULL = 0, OUT_UNITS = 1, OUT_LEAVES = 2, OUT_GROUPS = 3 };

struct GemmView {
  const void* A;
  int adt;
  int64_t lda;
  const void* B;
  int bdt;
  int64_t ldb;
  int64_t M, N, K;  // K = this view's extent (a rank shard or the whole K)
  int64_t bk, kf;   // numerics-defining plan (kf = global k_first)
  int64_t T, L;     // tiles in the view, leaf groups in the view (power of two)
};

struct GemmOut {
  int mode;            // OutMode
  int64_t tiles_per_unit;
  float* out;          // C (FULL) or workspace base
  int64_t ldo;         // row stride of C / of one workspace slice (= N)
  int64_t unit_stride; // elements between workspace slices
  uint16_t* act = nullptr;  // FULL only: write bf16(silu(gate) * up) of interleaved column pairs here
  int64_t ld_act = 0;       //   (row stride in elements; `out` is unused then)
  float* ms = nullptr;      // FULL only (tcgen05): also write the (m, s) state of every 16-column
  int64_t ld_ms = 0;        //   log-softmax chunk: ms[row][2 * (col / 16) + {0, 1}] (row stride ld_ms floats)
};

tbik_status launch_fma_gemm(const GemmView& v, const GemmOut& o, cudaStream_t s);
tbik_status launch_tc_gemm(const GemmView& v, const GemmOut& o, cudaStream_t s);
bool tc_supported(const GemmView& v, std::string* why);
// Output tiles of the tcgen05 kernel (one per CTA pair): 256 rows x 128 columns.
int64_t tc_pair_tiles(const GemmView& v);
// Work tiles of the variant launch_tc_gemm picks for v (pair 256 x 128 or single
// CTA 128 x 128) and how many run concurrently (CTA pairs or CTAs).
int64_t tc_tiles(const GemmView& v);
// Caps the SMs the tcgen05 GEMM's persistent grid may occupy on this host thread
// (0 = all); returns the previous cap.  Used to leave SMs for a concurrent
// all-reduce kernel (tbik_group.cu).
int set_tc_sm_cap(int cap);
int64_t tc_parallel_slots(const GemmView& v);

// Fused GEMM -> tree all-reduce (tbik_group.cu): while set on this host thread, a
// FULL-mode pair-tile launch_tc_gemm writes its partial into the group's send slot
// AND reduces the tiles this rank owns inside the same kernel (see
// tbik_gemm_tc.cu); `used` reports whether the launch took the fused path.
struct FusedAr {
  int W = 0, rank = 0;
  uint32_t epoch = 0;
  const float* src[8] = {};  // send slot of every rank (peer-mapped)
  float* dst[8] = {};        // result slot of every rank (peer-mapped)
  uint32_t* flags[8] = {};   // tile-flag array of every rank: [item][cta][W] u32
  uint32_t* done[8] = {};    // done[] of every rank
  uint32_t* counter = nullptr;
  int64_t flag_capacity = 0; // u32 words per tile-flag array
  bool used = false;
};
FusedAr* set_tc_fused_ar(FusedAr* ctx);

// Schedule overrides (tbik_set_schedule): how the work is cut and launched, never
// the per-element arithmetic.  Process-wide, set only through the C ABI (the
// library reads no environment variables).  knob() returns `dflt` when unset.
enum Knob {
  KNOB_TC_PAIR,          // 0/1: single-CTA 128x128 vs CTA-pair 256x128 tiles
  KNOB_TC_ABOX,          // 32/64/128: A rows staged per pipeline stage
  KNOB_TC_GROUP_M,       // raster: M blocks sharing one pass over W
  KNOB_TC_UNITS,         // K split of every output tile (power of two <= leaf groups)
  KNOB_TC_DEEP,          // 0/1: tree level 3 in scratch + deeper pipeline
  KNOB_TC_ACC4,          // 0: never four TMEM accumulators
  KNOB_TC_SKINNY,        // 0: no swap-AB kernel for M <= 128
  KNOB_SK_MT,            // skinny token tile 32/64/128
  KNOB_SK_UNITS,         // skinny K units
  KNOB_SK_LEAF,          // 1: skinny single-leaf units
  KNOB_SK_BN,            // skinny weight tile 32/64/128
  KNOB_FMA_V1,           // 1: the first FMA-leaf kernel
  KNOB_GROUP_FUSED,      // 0: no fused GEMM + all-reduce kernel
  KNOB_GROUP_OVERLAP,    // 0: no chunked GEMM / all-reduce overlap
  KNOB_AR_TWO_PHASE_BYTES,  // payload bytes from which the group all-reduce is two-phase
  KNOB_TC_WIDE,          // 0: 256 x 128 tiles, 1: 256 x 192 tiles (tbik_gemm_tc_w192.cu)
  KNOB_TC_WIDE_TAIL,     // 0: no half items in the wide kernels' last wave
  KNOB_SK_KS,            // skinny K rows per stage / W box: 64 or 128
  KNOB_SK_PDL,           // 0: skinny kernel without programmatic dependent launch
  KNOB_SK_TRACE,         // 1: skinny phase clocks to stderr (diagnostics)
  KNOB_SK_PAIR,          // 0: no CTA-pair split of a single leaf group (skinny)
  KNOB_ATTN_SV1,         // 0: tensor-core attention with double-buffered V (A/B)
  KNOB_ATTN_TC5,         // 1: tcgen05 attention form (tbik_attn_tc5.cu)
  KNOB_TC_PDL,           // 0: pair-tile GEMMs without programmatic dependent launch
  KNOB_COUNT
};
int64_t knob(Knob k, int64_t dflt);

tbik_status launch_tree_combine(const float* ws, int64_t X, int64_t fold, int64_t rows,
                                int64_t cols, float* out, int64_t ldo, cudaStream_t s);
tbik_status launch_allreduce(const PartPtrs& parts, int W, float* out, int64_t elems, bool ring,
                             bool aligned16, cudaStream_t s);

// Copies a bf16 operand whose row stride or base is not 16-byte aligned into a
// padded buffer (workspace slot `slot`); no-op otherwise.
tbik_status pad_operand(const void** p, int64_t* ld, int64_t rows, int64_t cols, int slot, cudaStream_t s);

// bf16(silu(gate) * up) over an f32 [rows x 2*inter] matrix whose columns
// interleave gate_j (2j) and up_j (2j+1) (tbik_model.cu).
tbik_status launch_silu_mul_il(const float* gu, int64_t ld, int64_t rows, int64_t inter, uint16_t* out, int64_t ldo,
                               cudaStream_t s);

// Swap-AB tcgen05 kernel for skinny views (M <= 64; tbik_gemm_skinny.cu): the
// whole tree (units finished in-kernel) into C.  Same bits as launch_tc_gemm.
bool tc_use_skinny(const GemmView& v);
tbik_status launch_tc_skinny(const GemmView& v, float* C, int64_t ldc, cudaStream_t s);

// 256 x 192 pair-tile variant of launch_tc_gemm (tbik_gemm_tc_w192.cu): FULL / UNITS
// modes without epilogues; same bits as the 256 x 128 kernel.
bool tc_wide_supported(const GemmView& v, const GemmOut& o);
// 0: the 256 x 128 kernel, 1: 256 x 192 tiles; knob tc_wide overrides.
int tc_wide_variant(const GemmView& v);
// K-split units the 256 x 192 kernel wants for v by default (1 or 2), 0 when it is
// not the default kernel for v.
int64_t tc_w192_units(const GemmView& v);
tbik_status launch_tc_w192(const GemmView& v, const GemmOut& o, cudaStream_t s);

// K-split factor run_tree_gemm uses for the tcgen05 leaf (1 = one FULL launch).
int64_t tc_split_units(const GemmView& v);

// View of A[M x K] . B[K x N] with the local plan of K under the given (global)
// k_first and c_max = 1 (matmul.cpp:153 via layers.cpp:85-88).
tbik_status make_view(const void* A, int adt, int64_t lda, const void* B, int bdt, int64_t ldb, int64_t M,
                      int64_t N, int64_t K, int64_t bk, int64_t kf_global, GemmView* v);

// Whole tree GEMM (plan resolved by the caller): picks FULL vs split + combine.
tbik_status run_tree_gemm(const GemmView& v, float* C, int64_t ldc, int leaf_mode, cudaStream_t s);

}  // namespace tbik_b200

namespace tbik_b200 {
// Per-CTA wait-cycle counters of the last tcgen05 launch (TBIK_TC_STATS=1).
int tc_debug_stats(unsigned long long* out, int max);
}  // namespace tbik_b200
