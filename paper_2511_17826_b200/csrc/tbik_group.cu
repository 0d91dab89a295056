// tbik_group.cu -- DeviceGroup (collective.hpp:15-23) with one process per
// GPU: the fixed-order tree all-reduce over NVLink peer memory.
//
// Each rank allocates one device region { send buffers [2][capacity] f32,
// flags [W] u32 } and exports it with CUDA IPC; every rank maps every peer's
// region.  A collective with epoch e (host counter, starts at 1):
//   1. the rank's partial is in its send buffer slot (e & 1) (the row-parallel
//      GEMM writes it there directly; otherwise one D2D copy);
//   2. the kernel's first CTA publishes "epoch e ready" into flags[rank] of
//      EVERY peer (st.release.sys after __threadfence_system), then every CTA
//      waits until its own flags[0..W) all reach e (ld.acquire.sys);
//   3. every rank reduces all W slots (e & 1) in Algorithm-2 order
//      (collective.cpp:67-74) straight from peer memory into its output.
// Double buffering + the per-collective barrier make slot reuse safe: a peer
// that publishes epoch e+1 has finished reading epoch e's slot.
// The sum order is per element and fixed, so all ranks produce identical
// bits -- the rank-symmetry the reference asserts (collective.cpp:79-85).
// NCCL / NVLS in-switch reduction are never used for the sum (order not
// controllable); NCCL appears only in bench.py's labelled baseline.
#include <cuda_runtime.h>

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

size_t flags_offset(int64_t capacity) { return static_cast<size_t>(2 * capacity) * sizeof(float); }

float* slot_ptr(char* region, int64_t capacity, uint32_t epoch) {
  return reinterpret_cast<float*>(region) + static_cast<size_t>(epoch & 1u) * capacity;
}

struct GroupPtrs {
  const float* src[kMaxRanks];
  uint32_t* flags[kMaxRanks];  // flags array of every rank (peer-mapped)
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void group_allreduce_kernel(GroupPtrs g, int W, int rank, uint32_t epoch, int64_t elems,
                                       float* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x < W) {
    __threadfence_system();
    st_release_sys(g.flags[threadIdx.x] + rank, epoch);
  }
  if (threadIdx.x == 0) {
    const uint32_t* mine = g.flags[rank];
    for (int r = 0; r < W; ++r)
      while (static_cast<int32_t>(ld_acquire_sys(mine + r) - epoch) < 0) {
      }
  }
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n4 = elems / 4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 r[kMaxRanks <= 8 ? 8 : 8];
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
    reinterpret_cast<float4*>(out)[i] = r[0];
  }
  for (int64_t e = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < elems; e += stride) {
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
    out[e] = r[0];
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
  g->region_bytes = flags_offset(capacity_elems) + 256;
  cudaError_t e = cudaMalloc(&g->region, g->region_bytes);
  if (e != cudaSuccess) {
    delete g;
    return cuda_status(e, "cudaMalloc(group region)");
  }
  e = cudaMemset(g->region + flags_offset(capacity_elems), 0, 256);
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
  for (int r = 0; r < g->W; ++r)
    if (g->opened[r]) cudaIpcCloseMemHandle(g->peer_region[r]);
  cudaFree(g->region);
  delete g;
  return TBIK_OK;
}

float* tbik_group_send_buffer(tbik_group* g) {
  if (!g) return nullptr;
  return slot_ptr(g->region, g->capacity, g->epoch + 1);
}

tbik_status tbik_group_tree_all_reduce(tbik_group* g, const float* partial, float* out, int64_t elems, void* stream) {
  if (!g || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (elems < 0 || elems > g->capacity) return set_error(TBIK_COLLECTIVE_MISMATCH, "elems exceed group capacity");
  for (int r = 0; r < g->W; ++r)
    if (!g->peer_region[r]) return set_error(TBIK_COLLECTIVE_MISMATCH, "peers not opened");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t epoch = ++g->epoch;
  float* mine = slot_ptr(g->region, g->capacity, epoch);
  if (partial && partial != mine)
    TBIK_CUDA(cudaMemcpyAsync(mine, partial, elems * sizeof(float), cudaMemcpyDeviceToDevice, s));
  GroupPtrs gp{};
  for (int r = 0; r < g->W; ++r) {
    gp.src[r] = slot_ptr(g->peer_region[r], g->capacity, epoch);
    gp.flags[r] = reinterpret_cast<uint32_t*>(g->peer_region[r] + flags_offset(g->capacity));
  }
  int64_t blocks = (elems / 4 + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  // All CTAs spin on the flags, so the grid must be co-resident: <= 4 per SM.
  group_allreduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(gp, g->W, g->rank, epoch, elems, out);
  TBIK_CUDA(cudaGetLastError());
  count_launch();
  return TBIK_OK;
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
  // GEMM straight into the peer-visible slot of the coming epoch.
  float* send = tbik_group_send_buffer(g);
  TBIK_TRY(tbik_tree_matmul(X_shard, x_dtype, ldx, W_shard, w_dtype, ldw, send, N, M, N, Kr, &local, leaf_mode,
                            stream));
  return tbik_group_tree_all_reduce(g, send, Y, M * N, stream);
}

}  // extern "C"
