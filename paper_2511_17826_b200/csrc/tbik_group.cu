// tbik_group.cu -- DeviceGroup (collective.hpp:15-23) with one process per
// GPU: the fixed-order tree all-reduce over NVLink peer memory.
//
// Each rank allocates one device region
//   { send [2][capacity] f32, result [2][capacity] f32, control block }
// and exports it with CUDA IPC; every rank maps every peer's region.  A
// collective with epoch e (host counter, starts at 1):
//   1. the rank's partial is in its send slot (e & 1) (the row-parallel GEMM
//      writes it there directly; otherwise one D2D copy);
//   2. barrier A: the kernel publishes "epoch e ready" into ready[rank] of EVERY
//      peer (st.release.sys after __threadfence_system), then waits until its
//      own ready[0..W) all reach e (ld.acquire.sys);
//   3a. small payloads (one-shot): every rank reduces all W slots in
//      Algorithm-2 order (collective.cpp:67-74) straight from peer memory into
//      its output -- one kernel, one barrier, W-1 remote reads per element;
//   3b. large payloads (reduce-scatter + push all-gather): rank r reduces only
//      element slice r (W-1 remote reads per element of the slice) and STORES
//      the reduced slice into the result slot (e & 1) of every rank over
//      NVLink; the last CTA to finish publishes done[rank] = e to every peer
//      (barrier B), and a second kernel waits for all W done flags and copies
//      the local result slot into the caller's output.  Per rank this moves
//      (W-1)/W of the payload in each NVLink direction instead of (W-1)x in.
// The per-element order is the same in 3a and 3b (Algorithm 2 over ranks
// 0..W-1), so every rank, every path and every schedule give identical bits:
// the rank symmetry the reference asserts (collective.cpp:79-85).
// Slot reuse is safe: a peer reaches epoch e+2 (same parity) only after
// barrier A of e+1, which every rank enters only after finishing epoch e.
// NCCL / NVLS in-switch reduction are never used for the sum (order not
// controllable); NCCL appears only in bench.py's labelled baseline.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "tbik_common.cuh"
#include "tbik_internal.h"

struct tbik_group {
  int W = 0, rank = 0, device = 0;
  int64_t capacity = 0;
  char* region = nullptr;  // own allocation
  size_t region_bytes = 0;
  char* peer_region[tbik_b200::kMaxRanks] = {};
  bool opened[tbik_b200::kMaxRanks] = {};
  uint32_t epoch = 0;
  int64_t fused = 0;  // row-parallel forwards that took the fused GEMM + all-reduce kernel
  // GEMM / all-reduce overlap (tbik_group_row_parallel_forward): a side stream for
  // the collectives and its events, created on first use.
  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_gemm = nullptr, ev_ar[2] = {nullptr, nullptr};
};

namespace tbik_b200 {
namespace {

constexpr int kHandleMagic = 0x5442494B;  // "TBIK"

struct HandleBlob {
  cudaIpcMemHandle_t h;  // 64 bytes
  int32_t magic;
  int32_t rank;
  int32_t world;
  int32_t device;
  int64_t capacity;
  char pad[TBIK_IPC_HANDLE_BYTES - 64 - 24];
};
static_assert(sizeof(HandleBlob) == TBIK_IPC_HANDLE_BYTES, "handle blob size");

// Control block after the four slots: ready[64] u32, done[64] u32, counter u32.
constexpr size_t kCtlBytes = 1024;
size_t flags_offset(int64_t capacity) { return static_cast<size_t>(4 * capacity) * sizeof(float); }
uint32_t* ready_flags(char* region, int64_t capacity) {
  return reinterpret_cast<uint32_t*>(region + flags_offset(capacity));
}
uint32_t* done_flags(char* region, int64_t capacity) { return ready_flags(region, capacity) + 64; }
uint32_t* cta_counter(char* region, int64_t capacity) { return ready_flags(region, capacity) + 128; }
uint32_t* fused_counter(char* region, int64_t capacity) { return ready_flags(region, capacity) + 129; }
// Tile flags of the fused GEMM -> all-reduce, after the control block:
// [item][cta of the pair][source rank] u32 (an item is a 256 x 128 output tile).
int64_t tile_flag_words(int64_t capacity, int W) { return 2 * int64_t(W) * (capacity / (256 * 128) + 1024); }
uint32_t* tile_flags(char* region, int64_t capacity) {
  return reinterpret_cast<uint32_t*>(region + flags_offset(capacity) + 1024);
}
float* result_ptr(char* region, int64_t capacity, uint32_t epoch) {
  return reinterpret_cast<float*>(region) + static_cast<size_t>(2 + (epoch & 1u)) * capacity;
}
// Payloads at or above this many bytes take the reduce-scatter + push path.
constexpr int64_t kTwoPhaseBytes = int64_t(1) << 20;

float* slot_ptr(char* region, int64_t capacity, uint32_t epoch) {
  return reinterpret_cast<float*>(region) + static_cast<size_t>(epoch & 1u) * capacity;
}

struct GroupPtrs {
  const float* src[8];   // send slot (e & 1) of every rank (peer-mapped)
  float* dst[8];         // result slot (e & 1) of every rank (peer-mapped)
  uint32_t* flags[8];    // ready[] array of every rank (peer-mapped)
  uint32_t* done[8];     // done[] array of every rank (peer-mapped)
};

// Barrier A: publish "epoch ready" to every peer (block 0), wait for all W.
__device__ __forceinline__ void barrier_ready(const GroupPtrs& g, int W, int rank, uint32_t epoch) {
  if (blockIdx.x == 0 && threadIdx.x < W) {
    __threadfence_system();
    st_release_sys(g.flags[threadIdx.x] + rank, epoch);
  }
  if (threadIdx.x == 0) {
    const uint32_t* mine = g.flags[rank];
    for (int r = 0; r < W; ++r) spin_until_epoch(mine + r, epoch);
  }
  __syncthreads();
}

// Algorithm 2 (collective.cpp:67-74) over the W rank values of one float4:
// for l = 1..log2 W, R[left] += R[left + 2^(l-1)] at every left step 2^l.
__device__ __forceinline__ float4 tree4(const GroupPtrs& g, int W, int64_t i) {
  float4 r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (k < W) r[k] = reinterpret_cast<const float4*>(g.src[k])[i];
#pragma unroll
  for (int l = 1; l <= 3; ++l) {
    const int st = 1 << l, h = 1 << (l - 1);
#pragma unroll
    for (int left = 0; left < 8; left += st)
      if (left + h < W) {
        r[left].x = __fadd_rn(r[left].x, r[left + h].x);
        r[left].y = __fadd_rn(r[left].y, r[left + h].y);
        r[left].z = __fadd_rn(r[left].z, r[left + h].z);
        r[left].w = __fadd_rn(r[left].w, r[left + h].w);
      }
  }
  return r[0];
}

__device__ __forceinline__ float tree1(const GroupPtrs& g, int W, int64_t e) {
  float r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (k < W) r[k] = g.src[k][e];
#pragma unroll
  for (int l = 1; l <= 3; ++l) {
    const int st = 1 << l, h = 1 << (l - 1);
#pragma unroll
    for (int left = 0; left < 8; left += st)
      if (left + h < W) r[left] = __fadd_rn(r[left], r[left + h]);
  }
  return r[0];
}

// 3a: one-shot -- every rank reduces every element.
__global__ void group_allreduce_kernel(GroupPtrs g, int W, int rank, uint32_t epoch, int64_t elems,
                                       float* __restrict__ out) {
  barrier_ready(g, W, rank, epoch);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n4 = elems / 4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride)
    reinterpret_cast<float4*>(out)[i] = tree4(g, W, i);
  for (int64_t e = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < elems; e += stride)
    out[e] = tree1(g, W, e);
}

// 3b, phase 1: reduce slice `rank` (float4 units [lo, hi)) and push it into
// every rank's result slot; the last CTA publishes done[rank] = epoch to all.
__global__ void group_reduce_scatter_push_kernel(GroupPtrs g, int W, int rank, uint32_t epoch, int64_t lo,
                                                 int64_t hi, uint32_t* __restrict__ counter) {
  barrier_ready(g, W, rank, epoch);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = lo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < hi; i += stride) {
    const float4 v = tree4(g, W, i);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < W) reinterpret_cast<float4*>(g.dst[(rank + k) & (W - 1)])[i] = v;  // stagger the peers
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(counter, 1u);
    if (prev == gridDim.x - 1) {
      *counter = 0;  // the next epoch's kernel starts after this one (stream order)
      __threadfence_system();
      for (int r = 0; r < W; ++r) st_release_sys(g.done[r] + rank, epoch);
    }
  }
}

// 3b, phase 2: wait until every rank has pushed its slice, then copy the local
// result slot into the caller's output.
__global__ void group_gather_wait_copy_kernel(const uint32_t* done, int W, uint32_t epoch,
                                              const float* __restrict__ result, float* __restrict__ out,
                                              int64_t elems) {
  if (threadIdx.x == 0)
    for (int r = 0; r < W; ++r) spin_until_epoch(done + r, epoch);
  __syncthreads();
  if (result == out) return;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    for (int64_t i = t0; i < elems / 4; i += stride)
      reinterpret_cast<float4*>(out)[i] = reinterpret_cast<const float4*>(result)[i];
  } else {
    for (int64_t i = t0; i < elems; i += stride) out[i] = result[i];
  }
}

// Barrier A alone (one CTA): used by the collectives whose consumer kernel is a
// plain launcher reading the peers' send slots (all-gather, (m, s) merge).
__global__ void group_barrier_kernel(GroupPtrs g, int W, int rank, uint32_t epoch) {
  barrier_ready(g, W, rank, epoch);
}

// All-gather (collective.cpp:46-50, layers.cpp:61-70): rank q's block sits dense
// in its send slot ([rows][row_units] of U); out[row][q * row_units + j] = it.
// blockIdx.y = source rank (staggered: rank r starts with r+1, own block last,
// so the W-1 NVLink reads of a step go to W-1 different peers).
template <typename U>
__global__ void group_gather_copy_kernel(GroupPtrs g, int W, int rank, int64_t rows, int64_t row_units,
                                         U* __restrict__ out, int64_t ld_out_units) {
  const int q = (rank + 1 + static_cast<int>(blockIdx.y)) & (W - 1);
  const U* __restrict__ src = reinterpret_cast<const U*>(g.src[q]);
  U* dst = out + static_cast<int64_t>(q) * row_units;
  const int64_t n = rows * row_units;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / row_units, c = i - r * row_units;
    dst[r * ld_out_units + c] = __ldcg(src + i);  // L2 / NVLink, never a stale L1 line
  }
}

}  // namespace
}  // namespace tbik_b200

using namespace tbik_b200;

extern "C" {

tbik_status tbik_group_create(int world_size, int rank, int device, int64_t capacity_elems, tbik_group** out) {
  if (!out) return set_error(TBIK_BAD_ARGUMENT, "null out");
  if (world_size < 1 || (world_size & (world_size - 1)))
    return set_error(TBIK_BAD_WORLD_SIZE, "world size must be a power of two, got " + std::to_string(world_size));
  if (world_size > 8) return set_error(TBIK_BAD_WORLD_SIZE, "peer group supports up to 8 ranks (one NVLink domain)");
  if (rank < 0 || rank >= world_size) return set_error(TBIK_BAD_ARGUMENT, "rank out of range");
  if (capacity_elems < 1 || capacity_elems % 4) return set_error(TBIK_BAD_ARGUMENT, "capacity must be a positive multiple of 4");
  TBIK_CUDA(cudaSetDevice(device));
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device");
  tbik_group* g = new tbik_group();
  g->W = world_size;
  g->rank = rank;
  g->device = device;
  g->capacity = capacity_elems;
  g->region_bytes = flags_offset(capacity_elems) + kCtlBytes + tile_flag_words(capacity_elems, world_size) * 4;
  cudaError_t e = cudaMalloc(&g->region, g->region_bytes);
  if (e != cudaSuccess) {
    delete g;
    return cuda_status(e, "cudaMalloc(group region)");
  }
  e = cudaMemset(g->region + flags_offset(capacity_elems), 0, g->region_bytes - flags_offset(capacity_elems));
  if (e != cudaSuccess) {
    cudaFree(g->region);
    delete g;
    return cuda_status(e, "cudaMemset(flags)");
  }
  g->peer_region[rank] = g->region;
  *out = g;
  return TBIK_OK;
}

tbik_status tbik_group_ipc_handle(tbik_group* g, void* handle_out) {
  if (!g || !handle_out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  HandleBlob b;
  std::memset(&b, 0, sizeof(b));
  TBIK_CUDA(cudaSetDevice(g->device));
  TBIK_CUDA(cudaIpcGetMemHandle(&b.h, g->region));
  b.magic = kHandleMagic;
  b.rank = g->rank;
  b.world = g->W;
  b.device = g->device;
  b.capacity = g->capacity;
  std::memcpy(handle_out, &b, sizeof(b));
  return TBIK_OK;
}

tbik_status tbik_group_open_peers(tbik_group* g, const void* handles) {
  if (!g || !handles) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  TBIK_CUDA(cudaSetDevice(g->device));
  for (int r = 0; r < g->W; ++r) {
    HandleBlob b;
    std::memcpy(&b, static_cast<const char*>(handles) + r * TBIK_IPC_HANDLE_BYTES, sizeof(b));
    if (b.magic != kHandleMagic || b.rank != r || b.world != g->W || b.capacity != g->capacity)
      return set_error(TBIK_COLLECTIVE_MISMATCH, "rank " + std::to_string(r) + " handle does not match this group");
    if (r == g->rank) continue;
    void* p = nullptr;
    TBIK_CUDA(cudaIpcOpenMemHandle(&p, b.h, cudaIpcMemLazyEnablePeerAccess));
    g->peer_region[r] = static_cast<char*>(p);
    g->opened[r] = true;
  }
  return TBIK_OK;
}

tbik_status tbik_group_destroy(tbik_group* g) {
  if (!g) return TBIK_OK;
  cudaSetDevice(g->device);
  cudaDeviceSynchronize();
  if (g->side) {
    cudaStreamDestroy(g->side);
    cudaEventDestroy(g->ev_start);
    cudaEventDestroy(g->ev_gemm);
    cudaEventDestroy(g->ev_ar[0]);
    cudaEventDestroy(g->ev_ar[1]);
  }
  for (int r = 0; r < g->W; ++r)
    if (g->opened[r]) cudaIpcCloseMemHandle(g->peer_region[r]);
  cudaFree(g->region);
  delete g;
  return TBIK_OK;
}

int tbik_group_world_size(const tbik_group* g) { return g ? g->W : 0; }
int tbik_group_rank(const tbik_group* g) { return g ? g->rank : -1; }
int64_t tbik_group_fused_count(const tbik_group* g) { return g ? g->fused : 0; }

float* tbik_group_send_buffer(tbik_group* g) {
  if (!g) return nullptr;
  return slot_ptr(g->region, g->capacity, g->epoch + 1);
}

namespace {
// max_blocks > 0 bounds every collective kernel's grid (the CTAs that can run
// beside a GEMM occupying the other SMs).
tbik_status check_group_operands(const void* X, int64_t ldx, const void* W, int64_t ldw, int64_t M, int64_t N,
                                 int64_t Kr) {
  if (!X || !W) return set_error(TBIK_BAD_ARGUMENT, "null operand");
  if (M < 1 || N < 1 || Kr < 1) return set_error(TBIK_BAD_DIMENSION, "dimensions must be >= 1");
  if (ldx < Kr || ldw < N) return set_error(TBIK_BAD_ARGUMENT, "leading dimension too small");
  return TBIK_OK;
}

GroupPtrs group_ptrs(tbik_group* g, uint32_t epoch) {
  GroupPtrs gp{};
  for (int r = 0; r < g->W; ++r) {
    gp.src[r] = slot_ptr(g->peer_region[r], g->capacity, epoch);
    gp.dst[r] = result_ptr(g->peer_region[r], g->capacity, epoch);
    gp.flags[r] = ready_flags(g->peer_region[r], g->capacity);
    gp.done[r] = done_flags(g->peer_region[r], g->capacity);
  }
  return gp;
}

// One "publish" epoch: this rank's `rows` x `row_bytes` block (row stride
// ld_bytes) is copied densely into its send slot, then barrier A.  Afterwards
// every peer's block of the same epoch is readable through *gp.  Slot reuse
// follows the epoch argument at the top of this file (a rank writes slot e & 1
// again only after barrier A of e+1, which every peer enters after its consumer
// of epoch e finished, in stream order).
tbik_status group_publish(tbik_group* g, const void* src, int64_t rows, int64_t row_bytes, int64_t ld_bytes,
                          cudaStream_t s, GroupPtrs* gp) {
  for (int r = 0; r < g->W; ++r)
    if (!g->peer_region[r]) return set_error(TBIK_COLLECTIVE_MISMATCH, "peers not opened");
  if (rows * row_bytes > g->capacity * static_cast<int64_t>(sizeof(float)))
    return set_error(TBIK_COLLECTIVE_MISMATCH, "block exceeds group capacity");
  const uint32_t epoch = ++g->epoch;
  void* mine = slot_ptr(g->region, g->capacity, epoch);
  if (rows > 0 && row_bytes > 0)
    TBIK_CUDA(cudaMemcpy2DAsync(mine, row_bytes, src, ld_bytes, row_bytes, rows, cudaMemcpyDeviceToDevice, s));
  *gp = group_ptrs(g, epoch);
  group_barrier_kernel<<<1, 32, 0, s>>>(*gp, g->W, g->rank, epoch);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}

// force_two_phase: the overlapped chunk pipeline reuses a send slot as soon as
// THIS rank's all-reduce of the slot finished, which proves every peer finished
// reading it only on the two-phase path (its done flags); it must not take the
// one-shot path whatever TBIK_AR_TWO_PHASE_BYTES says.
tbik_status group_all_reduce(tbik_group* g, const float* partial, float* out, int64_t elems, cudaStream_t s,
                             int64_t max_blocks, bool force_two_phase = false) {
  if (!g || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (elems < 0 || elems > g->capacity) return set_error(TBIK_COLLECTIVE_MISMATCH, "elems exceed group capacity");
  for (int r = 0; r < g->W; ++r)
    if (!g->peer_region[r]) return set_error(TBIK_COLLECTIVE_MISMATCH, "peers not opened");
  const uint32_t epoch = ++g->epoch;
  float* mine = slot_ptr(g->region, g->capacity, epoch);
  if (partial && partial != mine)
    TBIK_CUDA(cudaMemcpyAsync(mine, partial, elems * sizeof(float), cudaMemcpyDeviceToDevice, s));
  GroupPtrs gp{};
  for (int r = 0; r < g->W; ++r) {
    gp.src[r] = slot_ptr(g->peer_region[r], g->capacity, epoch);
    gp.dst[r] = result_ptr(g->peer_region[r], g->capacity, epoch);
    gp.flags[r] = ready_flags(g->peer_region[r], g->capacity);
    gp.done[r] = done_flags(g->peer_region[r], g->capacity);
  }
  const int64_t two_phase_bytes = knob(KNOB_AR_TWO_PHASE_BYTES, kTwoPhaseBytes);  // schedule only: same bits
  // The path must be the same on every rank: it depends only on (W, elems).
  if (g->W > 1 && elems % 4 == 0 && (force_two_phase || elems * 4 >= two_phase_bytes)) {
    const int64_t n4 = elems / 4;
    const int64_t lo = n4 * g->rank / g->W, hi = n4 * (g->rank + 1) / g->W;
    int64_t blocks = (hi - lo + 255) / 256;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, max_blocks > 0 ? max_blocks : 148 * 2));
    group_reduce_scatter_push_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
        gp, g->W, g->rank, epoch, lo, hi, cta_counter(g->region, g->capacity));
    TBIK_CUDA(cudaGetLastError());
    count_launch();
    int64_t cblocks = std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, max_blocks > 0 ? max_blocks : 148 * 4));
    group_gather_wait_copy_kernel<<<static_cast<unsigned>(cblocks), 256, 0, s>>>(
        done_flags(g->region, g->capacity), g->W, epoch, result_ptr(g->region, g->capacity, epoch), out, elems);
    TBIK_CUDA(cudaGetLastError());
    count_launch();
    return TBIK_OK;
  }
  int64_t blocks = (elems / 4 + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (max_blocks > 0 && blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  // All CTAs spin on the flags, so the grid must be co-resident: <= 4 per SM.
  group_allreduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(gp, g->W, g->rank, epoch, elems, out);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
}
}  // namespace

tbik_status tbik_group_tree_all_reduce(tbik_group* g, const float* partial, float* out, int64_t elems, void* stream) {
  return group_all_reduce(g, partial, out, elems, static_cast<cudaStream_t>(stream), 0);
}

tbik_status tbik_group_row_parallel_forward(tbik_group* g, const void* X_shard, int x_dtype, int64_t ldx,
                                            const void* W_shard, int w_dtype, int64_t ldw, float* Y, int64_t ldy,
                                            int64_t M, int64_t N, int64_t K_global, const tbik_block_config* cfg,
                                            int64_t c_max, int leaf_mode, void* stream) {
  if (!g || !cfg) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (ldy != N) return set_error(TBIK_BAD_ARGUMENT, "group row-parallel output must be dense (ldy == N)");
  if (M * N > g->capacity) return set_error(TBIK_COLLECTIVE_MISMATCH, "M*N exceeds group capacity");
  int64_t bounds[2 * kMaxRanks];
  TBIK_TRY(tbik_make_row_shard_plan(K_global, cfg, g->W, c_max, bounds));
  tbik_reduction_plan gp;
  TBIK_TRY(tbik_plan_blocks(K_global, cfg, c_max, &gp));
  const int64_t Kr = bounds[2 * g->rank + 1] - bounds[2 * g->rank];
  tbik_block_config local = *cfg;
  local.k_first = gp.k_first;  // layers.cpp:85-88
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t xsz = x_dtype == TBIK_BF16 ? 2 : 4;

  // Fused GEMM -> all-reduce (one kernel, tile by tile; schedule knob group_fused = 0 disables):
  // the tcgen05 GEMM writes its partial into this epoch's peer-visible send slot,
  // publishes every finished 256 x 128 tile to the tile's owner rank (item % W), and
  // warps 2-3 of every CTA reduce the tiles this rank owns in Algorithm-2 order
  // straight from the peers' slots and push the result into every rank's result
  // slot -- the NVLink traffic overlaps the tensor-core work of the same kernel.  A
  // short wait kernel then copies the result slot to Y once all W ranks are done.
  // Every rank must take the same path, so the choice uses only values that are
  // equal on every rank -- (M, N, leaf mode, W) -- never this rank's K range (the
  // last rank of a ragged K has fewer tiles, and the K-split / skinny heuristics
  // of tbik_tree_matmul look at it): M > 128 (pair tiles), N % 4 == 0 (TMA store).
  // The GEMM is then launched as ONE FULL-mode pair-tile launch on every rank.
  const bool fused_on = knob(KNOB_GROUP_FUSED, 1) != 0;
  if (fused_on && g->W > 1 && leaf_mode == TBIK_LEAF_TCGEN05 && M > 128 && N % 4 == 0 &&
      x_dtype == TBIK_BF16 && w_dtype == TBIK_BF16) {
    for (int r = 0; r < g->W; ++r)
      if (!g->peer_region[r]) return set_error(TBIK_COLLECTIVE_MISMATCH, "peers not opened");
    TBIK_TRY(check_group_operands(X_shard, ldx, W_shard, ldw, M, N, Kr));
    const uint32_t epoch = g->epoch + 1;
    FusedAr ar;
    ar.W = g->W;
    ar.rank = g->rank;
    ar.epoch = epoch;
    for (int r = 0; r < g->W; ++r) {
      ar.src[r] = slot_ptr(g->peer_region[r], g->capacity, epoch);
      ar.dst[r] = result_ptr(g->peer_region[r], g->capacity, epoch);
      ar.flags[r] = tile_flags(g->peer_region[r], g->capacity);
      ar.done[r] = done_flags(g->peer_region[r], g->capacity);
    }
    ar.counter = fused_counter(g->region, g->capacity);
    ar.flag_capacity = tile_flag_words(g->capacity, g->W);
    float* send = slot_ptr(g->region, g->capacity, epoch);
    GemmView v;
    TBIK_TRY(make_view(X_shard, x_dtype, ldx, W_shard, w_dtype, ldw, M, N, Kr, local.block_k, local.k_first, &v));
    FusedAr* prev = set_tc_fused_ar(&ar);
    const tbik_status st = launch_tc_gemm(v, GemmOut{OUT_FULL, v.T, send, N, 0}, s);
    set_tc_fused_ar(prev);
    TBIK_TRY(st);
    // launch_tc_gemm declines the fused form only for rank-uniform reasons (a grid
    // whose clusters cannot all be co-resident, an experiment knob): then every
    // rank has its partial in the send slot and runs the regular all-reduce.
    if (!ar.used) return group_all_reduce(g, send, Y, M * N, s, 0);
    g->epoch = epoch;
    ++g->fused;
    int64_t cblocks = std::max<int64_t>(1, std::min<int64_t>((M * N / 4 + 255) / 256, 148 * 4));
    group_gather_wait_copy_kernel<<<static_cast<unsigned>(cblocks), 256, 0, s>>>(
        done_flags(g->region, g->capacity), g->W, epoch, result_ptr(g->region, g->capacity, epoch), Y, M * N);
    TBIK_CUDA(cudaGetLastError());
    count_launch();
    return TBIK_OK;
  }

  // Overlap (GEMM -> all-reduce): rows in chunks; the GEMM of
  // chunk c+1 runs on all but kReserve SMs while the tree all-reduce of chunk c
  // runs beside it on a side stream.  Each chunk is one collective epoch whose
  // partial the GEMM writes straight into that epoch's peer-visible send slot;
  // the GEMM of chunk c+2 (same slot parity) waits for chunk c's all-reduce to
  // finish on this rank.  The chunk all-reduces are forced onto the two-phase
  // path, whose completion on this rank (all W done flags) proves that every
  // peer has finished READING this rank's slot -- the one-shot path proves only
  // that this rank finished reading the peers' slots.  Chunking rows never
  // changes bits (batch invariance), and every rank cuts the same chunks (they
  // depend only on M).  Schedule knob group_overlap = 0 disables it.
  const bool overlap_on = knob(KNOB_GROUP_OVERLAP, 1) != 0;
  constexpr int kChunks = 4, kReserve = 16;
  const bool overlap = overlap_on && g->W > 1 && M >= 2 * 256 && N % 4 == 0 && M * N * 4 >= (int64_t(8) << 20);
  if (!overlap) {
    // GEMM straight into the peer-visible slot of the coming epoch.
    float* send = tbik_group_send_buffer(g);
    TBIK_TRY(tbik_tree_matmul(X_shard, x_dtype, ldx, W_shard, w_dtype, ldw, send, N, M, N, Kr, &local, leaf_mode,
                              stream));
    return tbik_group_tree_all_reduce(g, send, Y, M * N, stream);
  }
  if (!g->side) {
    TBIK_CUDA(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
    TBIK_CUDA(cudaEventCreateWithFlags(&g->ev_start, cudaEventDisableTiming));
    TBIK_CUDA(cudaEventCreateWithFlags(&g->ev_gemm, cudaEventDisableTiming));
    TBIK_CUDA(cudaEventCreateWithFlags(&g->ev_ar[0], cudaEventDisableTiming));
    TBIK_CUDA(cudaEventCreateWithFlags(&g->ev_ar[1], cudaEventDisableTiming));
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
  const int64_t chunk = ((M + kChunks - 1) / kChunks + 255) / 256 * 256;
  TBIK_CUDA(cudaEventRecord(g->ev_start, s));
  TBIK_CUDA(cudaStreamWaitEvent(g->side, g->ev_start, 0));
  const uint32_t base = g->epoch;
  const int prev_cap = set_tc_sm_cap(sms - kReserve);
  tbik_status st = TBIK_OK;
  int64_t c = 0;
  for (int64_t r0 = 0; r0 < M && st == TBIK_OK; r0 += chunk, ++c) {
    const int64_t rows = std::min(chunk, M - r0);
    if (c >= 2 && (st = cudaStreamWaitEvent(s, g->ev_ar[c & 1], 0) == cudaSuccess ? TBIK_OK
                                                                                : set_error(TBIK_CUDA_ERROR, "wait")))
      break;
    float* send = slot_ptr(g->region, g->capacity, base + static_cast<uint32_t>(c) + 1);
    st = tbik_tree_matmul(static_cast<const char*>(X_shard) + r0 * ldx * xsz, x_dtype, ldx, W_shard, w_dtype, ldw,
                          send, N, rows, N, Kr, &local, leaf_mode, s);
    if (st != TBIK_OK) break;
    if (cudaEventRecord(g->ev_gemm, s) != cudaSuccess || cudaStreamWaitEvent(g->side, g->ev_gemm, 0) != cudaSuccess) {
      st = set_error(TBIK_CUDA_ERROR, "overlap event");
      break;
    }
    st = group_all_reduce(g, send, Y + r0 * N, rows * N, g->side, 4 * kReserve, /*force_two_phase=*/true);
    if (st == TBIK_OK && cudaEventRecord(g->ev_ar[c & 1], g->side) != cudaSuccess)
      st = set_error(TBIK_CUDA_ERROR, "overlap event");
  }
  set_tc_sm_cap(prev_cap);
  TBIK_TRY(st);
  TBIK_CUDA(cudaStreamWaitEvent(s, g->ev_ar[(c - 1) & 1], 0));
  return TBIK_OK;
}

tbik_status tbik_group_barrier(tbik_group* g, void* stream) {
  if (!g) return set_error(TBIK_BAD_ARGUMENT, "null group");
  GroupPtrs gp;
  return group_publish(g, nullptr, 0, 0, 0, static_cast<cudaStream_t>(stream), &gp);
}

tbik_status tbik_group_all_gather(tbik_group* g, const void* local, int64_t rows, int64_t cols, int64_t ld_local,
                                  int elem_bytes, void* out, int64_t ld_out, void* stream) {
  if (!g || !local || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (elem_bytes != 2 && elem_bytes != 4) return set_error(TBIK_UNKNOWN_DTYPE, "all_gather: element size must be 2 or 4");
  if (rows < 1 || cols < 1) return set_error(TBIK_BAD_DIMENSION, "all_gather: dimensions must be >= 1");
  if (ld_local < cols || ld_out < cols * g->W) return set_error(TBIK_BAD_ARGUMENT, "all_gather: leading dimension too small");
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t row_bytes = cols * elem_bytes;
  const int64_t max_rows = g->capacity * static_cast<int64_t>(sizeof(float)) / row_bytes;
  if (max_rows < 1) return set_error(TBIK_COLLECTIVE_MISMATCH, "all_gather: one row exceeds group capacity");
  // 16-byte units when every row start is 16-byte aligned, else 4- or 2-byte units
  // (a pure copy: the unit never changes the bytes).
  const uintptr_t ob = reinterpret_cast<uintptr_t>(out);
  const int64_t ldo_bytes = ld_out * elem_bytes;
  const int unit = (row_bytes % 16 == 0 && ob % 16 == 0 && ldo_bytes % 16 == 0)  ? 16
                   : (row_bytes % 4 == 0 && ob % 4 == 0 && ldo_bytes % 4 == 0) ? 4
                                                                                : 2;
  for (int64_t r0 = 0; r0 < rows; r0 += max_rows) {  // one epoch per chunk of rows (same chunks on every rank)
    const int64_t nr = std::min(max_rows, rows - r0);
    GroupPtrs gp;
    TBIK_TRY(group_publish(g, static_cast<const char*>(local) + r0 * ld_local * elem_bytes, nr, row_bytes,
                           ld_local * elem_bytes, s, &gp));
    const int64_t units = nr * row_bytes / unit;
    dim3 grid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((units + 255) / 256, 148 * 2 / g->W + 1))),
              static_cast<unsigned>(g->W));
    char* o = static_cast<char*>(out) + r0 * ldo_bytes;
    if (unit == 16)
      group_gather_copy_kernel<uint4><<<grid, 256, 0, s>>>(gp, g->W, g->rank, nr, row_bytes / 16,
                                                           reinterpret_cast<uint4*>(o), ldo_bytes / 16);
    else if (unit == 4)
      group_gather_copy_kernel<uint32_t><<<grid, 256, 0, s>>>(gp, g->W, g->rank, nr, row_bytes / 4,
                                                              reinterpret_cast<uint32_t*>(o), ldo_bytes / 4);
    else
      group_gather_copy_kernel<uint16_t><<<grid, 256, 0, s>>>(gp, g->W, g->rank, nr, row_bytes / 2,
                                                              reinterpret_cast<uint16_t*>(o), ldo_bytes / 2);
    TBIK_CUDA(cudaGetLastError());
    count_launch();
  }
  return TBIK_OK;
}

tbik_status tbik_group_logsoftmax_merge(tbik_group* g, const float* ms_local, int64_t rows, float* lse, void* stream) {
  if (!g || !ms_local || !lse) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (rows < 1) return set_error(TBIK_BAD_DIMENSION, "logsoftmax merge: rows must be >= 1");
  if (current_device_checked() < 0) return set_error(TBIK_NO_DEVICE, "no sm_100 device (no CPU fallback)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t max_rows = g->capacity / 2;
  for (int64_t r0 = 0; r0 < rows; r0 += max_rows) {
    const int64_t nr = std::min(max_rows, rows - r0);
    GroupPtrs gp;
    TBIK_TRY(group_publish(g, ms_local + 2 * r0, 1, nr * 2 * static_cast<int64_t>(sizeof(float)),
                           nr * 2 * static_cast<int64_t>(sizeof(float)), s, &gp));
    // The W shard states meet in rank order through the contiguous-halves tree --
    // the same merge tbik_tree_logsoftmax_local applies to simulated shards.
    TBIK_TRY(tbik_logsoftmax_merge(gp.src, g->W, nr, lse + r0, stream));
  }
  return TBIK_OK;
}

}  // extern "C"
