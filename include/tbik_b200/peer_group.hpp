// tbik_b200/peer_group.hpp -- C++ wrapper of the one-process-per-GPU group
// (tbik_group_* in tbik_b200.h): a DeviceGroup (collective.hpp:15-23) whose
// ranks are processes joined over NVLink peer memory.  Header-only, RAII.
//
//   tbik::PeerGroup g(W, rank, device, capacity);
//   auto mine = g.ipc_handle();                 // send to every rank (any transport)
//   g.open_peers(all_handles_rank_ordered);     // W * TBIK_IPC_HANDLE_BYTES bytes
//   g.row_parallel_forward(x_shard, w_shard, y, M, N, K_global, cfg);   // device pointers
//
// Device-pointer calls are asynchronous on `stream` (cudaStream_t as void*);
// failures throw tbik::TbikError like the rest of the API.
#pragma once

#include <cstdint>
#include <vector>

#include "tbik/errors.hpp"
#include "tbik/layers.hpp"
#include "tbik/matmul.hpp"
#include "tbik_b200.h"

namespace tbik {

class PeerGroup {
 public:
  PeerGroup(int world_size, int rank, int device, std::int64_t capacity_elems) {
    check_status(tbik_group_create(world_size, rank, device, capacity_elems, &g_));
  }
  ~PeerGroup() { tbik_group_destroy(g_); }
  PeerGroup(const PeerGroup&) = delete;
  PeerGroup& operator=(const PeerGroup&) = delete;

  int world_size() const { return tbik_group_world_size(g_); }
  int rank() const { return tbik_group_rank(g_); }
  tbik_group* native() const { return g_; }

  std::vector<unsigned char> ipc_handle() const {
    std::vector<unsigned char> h(TBIK_IPC_HANDLE_BYTES);
    check_status(tbik_group_ipc_handle(g_, h.data()));
    return h;
  }
  void open_peers(const std::vector<unsigned char>& rank_ordered_handles) {
    if (rank_ordered_handles.size() != static_cast<std::size_t>(TBIK_IPC_HANDLE_BYTES) * world_size())
      fail(ErrorCode::CollectiveMismatch, "open_peers: expected world_size handles");
    check_status(tbik_group_open_peers(g_, rank_ordered_handles.data()));
  }

  void barrier(void* stream = nullptr) { check_status(tbik_group_barrier(g_, stream)); }
  // tree_all_reduce (collective.hpp:38-39): Algorithm-2 order over the ranks.
  void tree_all_reduce(const float* partial, float* out, std::int64_t elems, void* stream = nullptr) {
    check_status(tbik_group_tree_all_reduce(g_, partial, out, elems, stream));
  }
  // row_parallel_forward (layers.hpp:43-45) for this rank's K shard.
  void row_parallel_forward(const void* x_shard, Dtype x_dtype, std::int64_t ldx, const void* w_shard, Dtype w_dtype,
                            std::int64_t ldw, float* y, std::int64_t M, std::int64_t N, std::int64_t K_global,
                            const BlockConfig& cfg, std::int64_t c_max = 8, Leaf leaf = Leaf::Tcgen05,
                            void* stream = nullptr) {
    const tbik_block_config c{cfg.block_m, cfg.block_k, cfg.block_n, cfg.k_first};
    check_status(tbik_group_row_parallel_forward(g_, x_shard, static_cast<int>(x_dtype), ldx, w_shard,
                                                 static_cast<int>(w_dtype), ldw, y, N, M, N, K_global, &c, c_max,
                                                 static_cast<int>(leaf), stream));
  }
  // all_gather (collective.hpp:27-28) as the column-parallel concatenation.
  void all_gather(const void* local, std::int64_t rows, std::int64_t cols, std::int64_t ld_local, Dtype dtype,
                  void* out, std::int64_t ld_out, void* stream = nullptr) {
    check_status(tbik_group_all_gather(g_, local, rows, cols, ld_local, dtype == Dtype::F32 ? 4 : 2, out, ld_out,
                                       stream));
  }
  // Cross-rank (m, s) merge of the vocab-sharded tree log-softmax.
  void logsoftmax_merge(const float* ms_local, std::int64_t rows, float* lse, void* stream = nullptr) {
    check_status(tbik_group_logsoftmax_merge(g_, ms_local, rows, lse, stream));
  }

 private:
  tbik_group* g_ = nullptr;
};

}  // namespace tbik
