/*
 * tbik_b200.h -- the C ABI of the B200-native TBIK library (libtbik_b200.so).
 *
 * Plain pointers and sizes only: no torch, no C++ types, no exceptions cross
 * this boundary.  Every entry point names the reference interface it replaces
 * (/root/reference/proj/include/tbik/..., file:line).  The C++ mirror of the
 * reference API (include/tbik_b200/tbik.hpp) is implemented on top of this
 * header, and so are the Python bindings used by tests/ and bench.py.
 *
 * Memory convention: unless stated otherwise, matrix arguments are DEVICE
 * pointers, row-major with an explicit leading dimension in elements
 * (the reference Matrix is row-major, matrix.hpp:18-24).  `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).  Kernels are
 * asynchronous; argument errors are returned synchronously, device faults
 * surface from the next call or tbik_sync().
 *
 * There is NO CPU fallback: without a usable sm_100 device every compute
 * entry point returns TBIK_NO_DEVICE.
 */
#ifndef TBIK_B200_H_
#define TBIK_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TBIK_API __attribute__((visibility("default")))
#else
#define TBIK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: 0 = ok, 1 + tbik::ErrorCode (errors.hpp:8-20) for the
 * reference's error kinds, >= 100 for device-side conditions.  The C++ shim
 * rethrows codes 1..11 as tbik::TbikError(ErrorCode) (errors.hpp:22-35). */
typedef enum tbik_status {
  TBIK_OK = 0,
  TBIK_BAD_DIMENSION = 1,       /* ErrorCode::BadDimension       */
  TBIK_SHAPE_MISMATCH = 2,      /* ErrorCode::ShapeMismatch      */
  TBIK_BAD_MAGIC = 3,           /* ErrorCode::BadMagic           */
  TBIK_TRUNCATED = 4,           /* ErrorCode::Truncated          */
  TBIK_UNKNOWN_DTYPE = 5,       /* ErrorCode::UnknownDtype       */
  TBIK_PLAN_INFEASIBLE = 6,     /* ErrorCode::PlanInfeasible     */
  TBIK_SHARD_ERROR = 7,         /* ErrorCode::ShardError         */
  TBIK_BAD_WORLD_SIZE = 8,      /* ErrorCode::BadWorldSize       */
  TBIK_COLLECTIVE_MISMATCH = 9, /* ErrorCode::CollectiveMismatch */
  TBIK_BAD_ARGUMENT = 10,       /* ErrorCode::BadArgument        */
  TBIK_IO = 11,                 /* ErrorCode::Io                 */
  TBIK_CUDA_ERROR = 100,        /* a CUDA runtime/driver call failed */
  TBIK_NO_DEVICE = 101,         /* no sm_100 device visible: no fallback */
  TBIK_UNSUPPORTED = 102        /* shape/dtype not supported by the requested kernel */
} tbik_status;

/* tbik::Dtype (matrix.hpp:20): storage type tag. */
typedef enum tbik_dtype { TBIK_F32 = 0, TBIK_BF16 = 1 } tbik_dtype;

/* Which computation forms a LEAF (one block_k tile dot product, matmul.cpp:69-75).
 *  TBIK_LEAF_FMA      CUDA-core ascending-k fma chain from +0: bit-exact with
 *                     the reference leaf_dot for every input.
 *  TBIK_LEAF_TCGEN05  tcgen05.mma (kind::f16, bf16 x bf16 -> f32 in TMEM),
 *                     block_k/16 MMAs from a zeroed accumulator.  Every merge
 *                     above the leaf is the reference's f32 tree, bit-exact;
 *                     the leaf itself is ulp-bounded against leaf_dot
 *                     (DESIGN.md section 3).  bf16 inputs, block_k % 64 == 0.
 * Both modes are TP- and batch-invariant: the per-element expression never
 * depends on M, on the N shard, on the TP size or on the launch schedule. */
typedef enum tbik_leaf_mode { TBIK_LEAF_FMA = 0, TBIK_LEAF_TCGEN05 = 1 } tbik_leaf_mode;

/* tbik::BlockConfig (matmul.hpp:18-25).  block_k and k_first define the
 * numerics; block_m / block_n are accepted for API parity and do not affect
 * bits (the GPU picks its own output tiling). */
typedef struct tbik_block_config {
  int64_t block_m;
  int64_t block_k;
  int64_t block_n;
  int64_t k_first; /* 0 = smallest feasible (plan_blocks) */
} tbik_block_config;

/* tbik::ReductionPlan (matmul.hpp:30-35). */
typedef struct tbik_reduction_plan {
  int64_t tiles_total;
  int64_t k_first;
  int64_t leaves;
  int64_t depth;
} tbik_reduction_plan;

TBIK_API const char* tbik_status_string(int status);
/* Detail text of the last error raised on the calling host thread. */
TBIK_API const char* tbik_last_error(void);
TBIK_API int tbik_version(void);
/* 1 if an sm_100 device is usable, else 0 (never falls back to the CPU). */
TBIK_API int tbik_device_available(void);
/* Block until all work queued by this library on `stream` finished; reports
 * any asynchronous device fault. */
TBIK_API tbik_status tbik_sync(void* stream);
/* Schedule overrides (tuning and the schedule-invariance tests): change HOW work
 * is cut and launched -- tile shapes, K splits, raster, pipeline depth, which
 * kernel variant, fused vs separate collectives -- never the per-element
 * arithmetic (every schedule is tested bit-identical).  Process-wide; the
 * library reads no environment variables.  Names: tc_pair, tc_abox, tc_group_m,
 * tc_units, tc_deep, tc_acc4, tc_skinny, sk_mt, sk_units, sk_leaf, sk_bn,
 * fma_v1, group_fused, group_overlap, ar_two_phase_bytes, tc_wide, tc_wide_tail,
 * sk_ks, sk_pdl, sk_trace (diagnostics: phase clocks to stderr), sk_pair, attn_sv1, attn_tc5, tc_pdl.
 * value < 0 unsets one knob, name NULL unsets all; an unknown name is TBIK_BAD_ARGUMENT.  Every rank
 * of a group must use the same group_* / ar_* settings. */
TBIK_API tbik_status tbik_set_schedule(const char* name, int64_t value);
/* Number of kernels this library has launched in this process (all devices).
 * bench.py reports the delta over its timed region as gpu_launches. */
TBIK_API uint64_t tbik_launch_count(void);
/* Name of the last tree-GEMM kernel this host thread launched (tc_tree_gemm_kernel,
 * tc_w192_tree_gemm_kernel, tc_skinny_kernel,
 * fma_tree_gemm_v2, ...); "" before the first.  Diagnostics: which schedule ran. */
TBIK_API const char* tbik_last_kernel(void);
/* Diagnostics: when TBIK_TC_STATS=1, the last tcgen05 GEMM launch records per-CTA
 * wait-cycle counters (8 per CTA: producer empty-wait, MMA tempty-wait, MMA
 * full-wait, merge tfull-wait, producer loop, merge loop, merge busy, unused);
 * copies up to `max` of them and returns how many exist. */
TBIK_API int tbik_debug_tc_stats(unsigned long long* out, int max);

/* ---- planner (host, pure integer functions) ---------------------------- */

/* default_block_config (matmul.cpp:11-14). */
TBIK_API tbik_status tbik_default_block_config(int dtype, tbik_block_config* out);
/* plan_blocks (matmul.hpp:42-43, matmul.cpp:24-67). */
TBIK_API tbik_status tbik_plan_blocks(int64_t K, const tbik_block_config* cfg, int64_t c_max,
                             tbik_reduction_plan* out);
/* make_row_shard_plan (layers.hpp:31-32, layers.cpp:23-46); bounds = 2*tp int64. */
TBIK_API tbik_status tbik_make_row_shard_plan(int64_t K, const tbik_block_config* cfg, int tp,
                                     int64_t c_max, int64_t* bounds);
/* make_column_shard_plan (layers.hpp:27, layers.cpp:9-21); bounds = 2*tp int64. */
TBIK_API tbik_status tbik_make_column_shard_plan(int64_t N, int tp, int64_t* bounds);

/* ---- the TBIK GEMM ------------------------------------------------------- */

/* tree_matmul (matmul.hpp:53, matmul.cpp:143-205) on device memory:
 *   C[M x N] (f32, ldc) = tree over K of A[M x K] (a_dtype, lda) . B[K x N] (b_dtype, ldb)
 * with the reduction plan plan_blocks(K, cfg, 1).  cfg->k_first must be the
 * GLOBAL k_first when this is one rank's shard (layers.cpp:85-88). */
TBIK_API tbik_status tbik_tree_matmul(const void* A, int a_dtype, int64_t lda, const void* B, int b_dtype,
                             int64_t ldb, float* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                             const tbik_block_config* cfg, int leaf_mode, void* stream);

/* The gate_up projection with SiLU(gate) * up fused (demo.cpp:171-174): B's 2*I
 * columns interleave gate_j (column 2j) and up_j (column 2j+1); the tree GEMM's
 * f32 values g feed act[M x I] (bf16, ld_act) = bf16(silu(g[2j]) * g[2j+1]) --
 * bit-identical to tbik_tree_matmul followed by the same SiLU*up (the epilogue
 * runs in the tcgen05 kernel when it can, otherwise through a workspace). */
TBIK_API tbik_status tbik_tree_matmul_silu_mul(const void* A, int a_dtype, int64_t lda, const void* B,
                                      int b_dtype, int64_t ldb, void* act, int64_t ld_act, int64_t M,
                                      int64_t I, int64_t K, const tbik_block_config* cfg, int leaf_mode,
                                      void* stream);

/* The lm_head projection with the log-softmax's first pass fused:
 * C [M x N] f32 logits = tree_matmul(A, B) as tbik_tree_matmul, and chunk_ms
 * [M x ld_chunks states] (>= groups * ceil(N / groups / 16) per row; 2 f32 each) = the (m, s) state of every 16-column
 * chunk of each vocab group, computed by the tcgen05 GEMM's epilogue on the f32
 * logits in registers (when the GEMM is one FULL launch and N / groups % 16 == 0;
 * otherwise by a pass over C -- the same bits).  Feed chunk_ms to
 * tbik_logsoftmax_shard_state_chunks. */
TBIK_API tbik_status tbik_tree_matmul_logits(const void* A, int a_dtype, int64_t lda, const void* B, int b_dtype,
                                             int64_t ldb, float* C, int64_t ldc, float* chunk_ms, int64_t ld_chunks,
                                             int64_t M, int64_t N, int64_t K, int64_t groups,
                                             const tbik_block_config* cfg, int leaf_mode, void* stream);

/* Debug / verification entry: write every leaf partial product P_t
 * (t = 0..tiles_total-1) to leaves[t][M][N] (f32, dense) using the given leaf
 * mode.  tests/ feed these to the CPU oracle's tree to check the tree logic
 * above a tcgen05 leaf bit-for-bit ("oracle tree over GPU leaves"). */
TBIK_API tbik_status tbik_tree_matmul_leaves(const void* A, int a_dtype, int64_t lda, const void* B,
                                    int b_dtype, int64_t ldb, float* leaves, int64_t M, int64_t N,
                                    int64_t K, const tbik_block_config* cfg, int leaf_mode,
                                    void* stream);

/* column_parallel_forward (layers.hpp:36-38, layers.cpp:48-72) on ONE device
 * with `tp` simulated ranks (the reference's in-process DeviceGroup): rank r
 * computes the N-columns [r*N/tp, (r+1)*N/tp) with the c_max=1 plan; outputs
 * are concatenated.  No cross-shard arithmetic. */
TBIK_API tbik_status tbik_column_parallel_forward_local(const void* X, int x_dtype, int64_t ldx,
                                               const void* W, int w_dtype, int64_t ldw, float* Y,
                                               int64_t ldy, int64_t M, int64_t N, int64_t K,
                                               int tp, const tbik_block_config* cfg,
                                               int leaf_mode, void* stream);

/* row_parallel_forward (layers.hpp:43-45, layers.cpp:74-98) on ONE device with
 * `tp` simulated ranks: rank r runs tbik_tree_matmul on its K range
 * (make_row_shard_plan) with the global k_first into its own f32 partial,
 * then the partials meet in tbik_tree_all_reduce_local.  Bit-identical for
 * every feasible tp (the reference's claim, runner.cpp:53-91). */
TBIK_API tbik_status tbik_row_parallel_forward_local(const void* X, int x_dtype, int64_t ldx,
                                            const void* W, int w_dtype, int64_t ldw, float* Y,
                                            int64_t ldy, int64_t M, int64_t N, int64_t K, int tp,
                                            const tbik_block_config* cfg, int64_t c_max,
                                            int leaf_mode, void* stream);

/* ---- the fixed-order tree all-reduce ------------------------------------ */

/* tree_all_reduce_per_rank (collective.hpp:33-34, collective.cpp:52-92) over W
 * f32 buffers that are all addressable from the current device (local or
 * peer-mapped): out[e] = Algorithm-2 order  R[left] += R[left + 2^(l-1)].
 * W must be a power of two (BadWorldSize, collective.cpp:11-16). */
TBIK_API tbik_status tbik_tree_all_reduce_local(const float* const* partials, int W, float* out,
                                       int64_t elems, void* stream);

/* ring_reduce_baseline (collective.hpp:43-44, collective.cpp:94-106): the
 * labelled non-invariant left-to-right stand-in, for divergence tests. */
TBIK_API tbik_status tbik_ring_reduce_local(const float* const* partials, int W, float* out,
                                   int64_t elems, void* stream);

/* leaf_dot (matmul.hpp:48, matmul.cpp:69-75) on the device: *out = ascending-k
 * fma chain from +0 over a[0..n) . b[0..n) (f32, device pointers), one thread. */
TBIK_API tbik_status tbik_leaf_dot(const float* a, const float* b, int64_t n, float* out, void* stream);

/* silu (demo.hpp:56, demo.cpp:36-45): out[i][j] = z / (1 + exp(-z)), z = x widened
 * to f32; exp is the library's shared polynomial. */
TBIK_API tbik_status tbik_silu(const void* x, int x_dtype, int64_t ldx, int64_t rows, int64_t cols, float* out,
                               int64_t ldo, void* stream);

/* ---- one process, several GPUs (the reference's DeviceGroup, collective.hpp:15-23) --
 * World size W, rank r runs on device_ids[r] (ranks may share a device).  Peer
 * access is enabled between the distinct devices; every rank gets its own
 * stream on its device and a group-owned f32 partial buffer there. */
typedef struct tbik_local_group tbik_local_group;
TBIK_API tbik_status tbik_local_group_create(int world_size, const int* device_ids, tbik_local_group** out);
TBIK_API tbik_status tbik_local_group_destroy(tbik_local_group* g);
TBIK_API int tbik_local_group_device(const tbik_local_group* g, int rank);
/* Rank r's stream (cudaStream_t on its device): inputs a caller uploads for rank
 * r must be complete or ordered on it. */
TBIK_API void* tbik_local_group_stream(const tbik_local_group* g, int rank);
/* row_parallel_forward (layers.cpp:74-98) across the group's devices: rank r's
 * X_shards[r] [M x K_r] (row stride ldx[r]) and W_shards[r] [K_r x N] (ldw[r])
 * live on its device, K_r = make_row_shard_plan(K_global)[r].  Each rank's tree
 * GEMM (global k_first) runs on its own device and stream; then rank 0's device
 * reduces the W partials over peer memory in Algorithm-2 order into Y (on rank
 * 0's device, ldy).  `stream` (rank 0's device) is ordered after the result. */
TBIK_API tbik_status tbik_local_group_row_parallel_forward(tbik_local_group* g, const void* const* X_shards,
                                                           int x_dtype, const int64_t* ldx,
                                                           const void* const* W_shards, int w_dtype,
                                                           const int64_t* ldw, float* Y, int64_t ldy, int64_t M,
                                                           int64_t N, int64_t K_global, const tbik_block_config* cfg,
                                                           int64_t c_max, int leaf_mode, void* stream);

/* ---- the labelled NON-INVARIANT status quo (collective.cpp:94-106, layers.cpp:100-121) --
 * cuBLAS GEMMs (f32 accumulate, summation order chosen by the library) and a
 * left-to-right ring sum / NCCL all-reduce: the baseline the price of
 * determinism is measured against.  Never used by the TBIK path. */
/* C[M x N] f32 = A . B with cuBLAS (bf16 or f32 operands, f32 accumulate). */
TBIK_API tbik_status tbik_baseline_gemm(const void* A, int a_dtype, int64_t lda, const void* B, int b_dtype,
                                        int64_t ldb, float* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                                        void* stream);
/* baseline_row_parallel_forward (layers.cpp:100-121) with `tp` simulated ranks on
 * one device: K % tp == 0 (ShardError otherwise), rank r's cuBLAS GEMM over
 * [r*K/tp, (r+1)*K/tp), then ring_reduce_baseline (left to right). */
TBIK_API tbik_status tbik_baseline_row_parallel_forward_local(const void* X, int x_dtype, int64_t ldx, const void* W,
                                                              int w_dtype, int64_t ldw, float* Y, int64_t ldy,
                                                              int64_t M, int64_t N, int64_t K, int tp, void* stream);
/* baseline_column_parallel_forward (layers.cpp:122-146): cuBLAS per column shard. */
TBIK_API tbik_status tbik_baseline_column_parallel_forward_local(const void* X, int x_dtype, int64_t ldx,
                                                                 const void* W, int w_dtype, int64_t ldw, float* Y,
                                                                 int64_t ldy, int64_t M, int64_t N, int64_t K, int tp,
                                                                 void* stream);
/* NCCL communicator for the baseline across processes (one per GPU). */
#define TBIK_NCCL_ID_BYTES 128
TBIK_API tbik_status tbik_nccl_unique_id(void* id_out /* TBIK_NCCL_ID_BYTES */);
TBIK_API tbik_status tbik_nccl_comm_create(int world_size, int rank, int device, const void* id, void** comm);
TBIK_API tbik_status tbik_nccl_comm_destroy(void* comm);
/* The status-quo row-parallel layer per rank (SURVEY 8(b) tbik_baseline_cublas_nccl):
 * cuBLAS GEMM of this rank's shard X_shard [M x K_r] . W_shard [K_r x N], then an
 * NCCL sum all-reduce into Y [M x N] (dense).  out_f32 = 1: f32 GEMM output and f32
 * all-reduce (the same bytes on the wire as the TBIK tree all-reduce); 0: bf16
 * output and bf16 all-reduce (what a serving stack does).  Y is f32 or bf16
 * accordingly.  The summation order is NCCL's: not TP-invariant. */
TBIK_API tbik_status tbik_baseline_cublas_nccl(void* comm, const void* X_shard, int x_dtype, int64_t ldx,
                                               const void* W_shard, int w_dtype, int64_t ldw, void* Y, int64_t M,
                                               int64_t N, int64_t K_shard, int out_f32, void* stream);

/* ---- one-process-per-GPU groups (NVLink peer memory) -------------------- */

/* A DeviceGroup (collective.hpp:15-23) whose ranks are processes, one per GPU.
 * Each rank owns a peer-visible f32 exchange buffer of `capacity_elems`
 * (x2 for double buffering) plus a flag array; handles are exchanged out of
 * band (e.g. torch.distributed all_gather_object) with tbik_group_ipc_handle /
 * tbik_group_open_peers.  The reduction order is per element and fixed, so the
 * result is bit-identical on every rank and for every schedule. */
typedef struct tbik_group tbik_group;
#define TBIK_IPC_HANDLE_BYTES 128

TBIK_API tbik_status tbik_group_create(int world_size, int rank, int device, int64_t capacity_elems,
                              tbik_group** out);
TBIK_API tbik_status tbik_group_ipc_handle(tbik_group* g, void* handle_out /* TBIK_IPC_HANDLE_BYTES */);
TBIK_API tbik_status tbik_group_open_peers(tbik_group* g, const void* handles /* W * HANDLE_BYTES */);
TBIK_API tbik_status tbik_group_destroy(tbik_group* g);
/* World size / rank of the group (0 / -1 for a null handle). */
TBIK_API int tbik_group_world_size(const tbik_group* g);
TBIK_API int tbik_group_rank(const tbik_group* g);
/* This rank's exchange buffer for the next collective (device pointer). */
TBIK_API float* tbik_group_send_buffer(tbik_group* g);
/* Diagnostics: how many row-parallel forwards of this group ran as ONE fused
 * kernel (tcgen05 GEMM + tile-flag tree all-reduce over peer memory). */
TBIK_API int64_t tbik_group_fused_count(const tbik_group* g);

/* tree_all_reduce over the group: `partial` (elems f32, may be the send
 * buffer itself) is published, all ranks meet on a device-side flag barrier,
 * and every rank reduces all W partials in Algorithm-2 order into `out`. */
TBIK_API tbik_status tbik_group_tree_all_reduce(tbik_group* g, const float* partial, float* out,
                                       int64_t elems, void* stream);

/* row_parallel_forward for this rank: X_shard [M x K_r], W_shard [K_r x N]
 * (this rank's make_row_shard_plan range of the global K), GEMM straight into
 * the peer-visible send buffer, then the tree all-reduce into Y. */
TBIK_API tbik_status tbik_group_row_parallel_forward(tbik_group* g, const void* X_shard, int x_dtype,
                                            int64_t ldx, const void* W_shard, int w_dtype,
                                            int64_t ldw, float* Y, int64_t ldy, int64_t M,
                                            int64_t N, int64_t K_global,
                                            const tbik_block_config* cfg, int64_t c_max,
                                            int leaf_mode, void* stream);

/* A group-wide barrier (one epoch, no payload): returns once enqueued; the
 * stream continues only after every rank reached it. */
TBIK_API tbik_status tbik_group_barrier(tbik_group* g, void* stream);

/* all_gather (collective.hpp:27-28, collective.cpp:46-50) as the column-parallel
 * concatenation (layers.cpp:61-70): rank q's [rows x cols] block (elem_bytes 2
 * for bf16, 4 for f32; row stride ld_local elements) lands in columns
 * [q*cols, (q+1)*cols) of out [rows x W*cols] (row stride ld_out) on EVERY rank.
 * Rank-indexed, never arrival-ordered; rows beyond the group capacity are moved
 * in several epochs (every rank must pass the same rows / cols). */
TBIK_API tbik_status tbik_group_all_gather(tbik_group* g, const void* local, int64_t rows, int64_t cols,
                                           int64_t ld_local, int elem_bytes, void* out, int64_t ld_out,
                                           void* stream);

/* Cross-rank step of the vocab-sharded tree log-softmax (tbik_logsoftmax_merge
 * over the group): this rank's ms_local [rows x 2] f32 (tbik_logsoftmax_shard_state
 * of its vocab shard) is exchanged -- 8 bytes per row -- and every rank merges
 * the W states in rank order with the contiguous-halves tree into lse[rows]
 * (bit-identical to tbik_tree_logsoftmax_local with tp = W simulated shards). */
TBIK_API tbik_status tbik_group_logsoftmax_merge(tbik_group* g, const float* ms_local, int64_t rows, float* lse,
                                                 void* stream);

/* ---- host-buffer entry points (the reference's Matrix in / Matrix out) ---- */

/* tree_matmul (matmul.hpp:53) with HOST activations A_host [M x K] and a HOST
 * f32 result C_host [M x N]; the weights B stay in device memory.  Rows are
 * streamed in chunks of `chunk_rows` (0 = default): the H2D copy of chunk i+1,
 * the GEMM of chunk i and the D2H copy of chunk i-1 overlap on three streams.
 * Bit-identical to tbik_tree_matmul on device buffers (batch invariance).
 * Returns once enqueued; `stream` is ordered after the last D2H copy
 * (tbik_sync(stream) waits).  Page-locked host buffers give full overlap. */
TBIK_API tbik_status tbik_tree_matmul_hostio(const void* A_host, int a_dtype, int64_t lda, const void* B,
                                    int b_dtype, int64_t ldb, float* C_host, int64_t ldc, int64_t M,
                                    int64_t N, int64_t K, const tbik_block_config* cfg, int leaf_mode,
                                    int64_t chunk_rows, void* stream);

/* tbik_group_row_parallel_forward with this rank's HOST X shard [M x K_shard]
 * (K_shard = its make_row_shard_plan range) and a HOST Y [M x N], same
 * pipeline; one collective epoch per row chunk (every rank must pass the same
 * M and chunk_rows). */
TBIK_API tbik_status tbik_group_row_parallel_forward_hostio(tbik_group* g, const void* X_host_shard,
                                                   int x_dtype, int64_t ldx, const void* W_shard,
                                                   int w_dtype, int64_t ldw, float* Y_host,
                                                   int64_t ldy, int64_t M, int64_t N, int64_t K_shard,
                                                   int64_t K_global, const tbik_block_config* cfg,
                                                   int64_t c_max, int leaf_mode, int64_t chunk_rows,
                                                   void* stream);

/* ---- the reference's TBIK matrix file (host only) ------------------------ */

/* matrix_write (matrix.hpp:86, matrix.cpp:211-233): "TBIK", u16 version 1,
 * u16 dtype (0 f32 / 1 bf16), u64 rows, u64 cols, little-endian row-major
 * payload from the host buffer `data`.  TBIK_IO on open/short-write failure. */
TBIK_API tbik_status tbik_matrix_write(const char* path, const void* data, int dtype, int64_t rows,
                              int64_t cols);
/* matrix_read (matrix.hpp:87, matrix.cpp:235-284) in two calls: the header,
 * then the payload into a host buffer of capacity_bytes.  Errors as the
 * reference: TBIK_IO, TBIK_TRUNCATED, TBIK_BAD_MAGIC, TBIK_UNKNOWN_DTYPE
 * (unknown version or dtype code). */
TBIK_API tbik_status tbik_matrix_read_header(const char* path, int* dtype, int64_t* rows, int64_t* cols);
TBIK_API tbik_status tbik_matrix_read(const char* path, void* out, int64_t capacity_bytes);

/* ---- tree-ordered reductions (NEW semantics) -------- */

/* rmsnorm (demo.hpp:53, demo.cpp:11-34) with the sum of squares in the
 * canonical lane tree (oracle/tbik_oracle.c tbo_tree_rmsnorm):
 * Y = (X * gamma) / sqrt(tree_sum(X^2) / cols + eps).  y_dtype f32 or bf16. */
TBIK_API tbik_status tbik_tree_rmsnorm(const void* X, int x_dtype, int64_t ldx, const float* gamma,
                              float eps, void* Y, int y_dtype, int64_t ldy, int64_t rows,
                              int64_t cols, void* stream);

/* Vocab-sharded tree log-softmax, step 1: the (m, s) state of every one of
 * `groups` contiguous vocab groups of this shard (logits [rows x v_local] f32:
 * 16-logit chunk states meeting by pairwise levels inside a group),
 * then merged over the shard's groups by the canonical tree.  ms_out is
 * rows x 2 f32 ({m, s} per row) -- 8 bytes per row to exchange. */
TBIK_API tbik_status tbik_logsoftmax_shard_state(const float* logits, int64_t ld, int64_t rows,
                                        int64_t v_local, int64_t groups, float* ms_out,
                                        void* stream);
/* The same step 1 from the (m, s) states of the logits' 16-column chunks
 * (chunk_ms rows x (groups * ceil(v_local / groups / 16)) x 2 f32, chunks restart at
 * every group), as written by tbik_tree_matmul_logits or tbik_logsoftmax_chunk_states:
 * the logits are not read again.  Same bits as tbik_logsoftmax_shard_state. */
TBIK_API tbik_status tbik_logsoftmax_shard_state_chunks(const float* chunk_ms, int64_t ld_chunks, int64_t rows,
                                                        int64_t v_local, int64_t groups, float* ms_out, void* stream);
/* The chunk states of a logit block (the non-fused producer); ld_chunks = states per
 * row of chunk_ms (>= groups * ceil(v_local / groups / 16)). */
TBIK_API tbik_status tbik_logsoftmax_chunk_states(const float* logits, int64_t ld, int64_t rows, int64_t v_local,
                                                  int64_t groups, float* chunk_ms, int64_t ld_chunks, void* stream);
/* Step 2: merge W shard states (rank order, contiguous-halves tree) into
 * lse[rows] = m + log(s).  W a power of two. */
TBIK_API tbik_status tbik_logsoftmax_merge(const float* const* ms_parts, int W, int64_t rows, float* lse,
                                  void* stream);
/* Step 3: logprobs[i][j] = logits[i][j] - lse[i] (optional, may be NULL) and
 * target_logprobs[i] = logits[i][targets[i] - v_offset] - lse[i] for targets
 * that fall in this shard (optional). */
TBIK_API tbik_status tbik_logsoftmax_finish(const float* logits, int64_t ld, int64_t rows, int64_t v_local,
                                   const float* lse, float* logprobs, int64_t ld_out,
                                   const int64_t* targets, int64_t v_offset,
                                   float* target_logprobs, void* stream);
/* Single-device convenience: all three steps with `tp` simulated vocab shards. */
TBIK_API tbik_status tbik_tree_logsoftmax_local(const float* logits, int64_t ld, int64_t rows, int64_t V,
                                       int64_t groups, int tp, float* lse, float* logprobs,
                                       int64_t ld_out, const int64_t* targets,
                                       float* target_logprobs, void* stream);

/* ---- per-token kernels of a TBIK decoder forward ----------
 * The reference's toy model (demo.cpp:164-241) has no attention / RoPE; these
 * complete a Llama / Qwen-shaped forward whose every element is a fixed,
 * shard-independent sequence of RN f32 ops (restated in oracle/tbik_oracle.c). */

/* out[i] = table[ids[i]] (bf16 rows of width H); BadArgument on an id >= V. */
TBIK_API tbik_status tbik_embedding(const void* table, int64_t V, int64_t H, const int64_t* ids, int64_t rows,
                                    void* out, void* stream);
/* Rotate-half RoPE on f32 columns [col0, col0 + heads*head_dim) of x, bf16 out;
 * cos/sin tables are f32 [max_pos][head_dim/2], positions int32 [rows]. */
TBIK_API tbik_status tbik_rope(const float* x, int64_t ldx, int64_t col0, int heads, int head_dim,
                               const int* positions, const float* cos_table, const float* sin_table,
                               void* out, int64_t ldo, int64_t rows, void* stream);
/* The attention inputs of one qkv projection in one launch: tbik_rope of the
 * n_q_heads q heads (columns [0, nq hd)) into q_out [rows][nq hd], of the
 * n_kv_heads k heads (the next nkv hd columns) into k_out [rows][nkv hd], and
 * tbik_cast_bf16 of v (the last nkv hd columns) into v_out -- the same bits as the
 * three calls.  head_dim % 8 == 0, 16-byte aligned f32 rows (ld % 4 == 0). */
TBIK_API tbik_status tbik_rope_qkv(const float* qkv, int64_t ld, int n_q_heads, int n_kv_heads, int head_dim,
                                   const int* positions, const float* cos_table, const float* sin_table,
                                   void* q_out, void* k_out, void* v_out, int64_t rows, void* stream);
/* storage_cast (demo.cpp:50-52): bf16_round of an f32 block. */
TBIK_API tbik_status tbik_cast_bf16(const float* x, int64_t ldx, int64_t rows, int64_t cols, void* out,
                                    int64_t ldo, void* stream);
/* Causal GQA prefill attention over `batch` sequences of seq_len tokens (rows are
 * sequence-major), head_dim 128, bf16 in / bf16 out: the exact two-pass order
 * (ascending-d fma scores, exact max, shared exp, ascending sums), restated by the
 * oracle bit for bit; seq_len <= 512. */
TBIK_API tbik_status tbik_attention_prefill(const void* q, int64_t ldq, const void* k, int64_t ldk,
                                            const void* v, int64_t ldv, int64_t batch, int seq_len,
                                            int n_q_heads, int n_kv_heads, int head_dim, float scale,
                                            void* out, int64_t ldo, void* stream);
/* The same attention in a tensor-core flash form (mma.sync bf16 scores and P.V,
 * online softmax over 64-key blocks from key 0): deterministic, bit-identical across
 * batch composition and head sharding, within a tolerance of the exact form. */
TBIK_API tbik_status tbik_attention_prefill_tc(const void* q, int64_t ldq, const void* k, int64_t ldk,
                                               const void* v, int64_t ldv, int64_t batch, int seq_len,
                                               int n_q_heads, int n_kv_heads, int head_dim, float scale,
                                               void* out, int64_t ldo, void* stream);
/* act = bf16(silu(gate) * up), gate = columns [0, inter), up = [inter, 2 inter)
 * of gate_up (f32) -- silu (demo.cpp:36-45) with the shared exp. */
TBIK_API tbik_status tbik_silu_mul(const float* gate_up, int64_t ld, int64_t rows, int64_t inter, void* out,
                                   int64_t ldo, void* stream);
/* h = bf16(h + f) in place (demo.cpp:216). */
TBIK_API tbik_status tbik_residual_add(void* h, int64_t ldh, const float* f, int64_t ldf, int64_t rows,
                                       int64_t cols, void* stream);
/* h = bf16(h + f) in place, then y = tree RMSNorm of the new h (bf16 -> bf16):
 * exactly tbik_residual_add followed by tbik_tree_rmsnorm, in one pass when the
 * rows are 16-byte aligned with cols % 8 == 0 and cols <= 8192. */
TBIK_API tbik_status tbik_residual_rmsnorm(void* h, int64_t ldh, const float* f, int64_t ldf, const float* gamma,
                                           float eps, void* y, int64_t ldy, int64_t rows, int64_t cols,
                                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TBIK_B200_H_ */
