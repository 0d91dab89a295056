// tbik/collective.hpp -- drop-in for proj/include/tbik/collective.hpp
// (collective.hpp:15-45).  A DeviceGroup of W ranks held by ONE process, as in
// the reference; on the B200 rank r runs on GPU devices()[r].  By default the
// ranks are spread over the visible sm_100 devices (rank r on device
// r % device_count), so DeviceGroup(8) spans eight GPUs of an HGX node and
// collapses to simulated ranks on one GPU elsewhere -- same bits either way.
// Cross-device partials meet in the fixed-order tree all-reduce over peer
// memory (NVLink).  For one process per GPU see tbik_b200/peer_group.hpp.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "tbik/matrix.hpp"

struct tbik_local_group;

namespace tbik {

class TBIK_CPP_API DeviceGroup {
 public:
  explicit DeviceGroup(int world_size);
  // B200 addition: explicit rank -> device map (devices.size() == world_size).
  DeviceGroup(int world_size, std::vector<int> devices);

  int world_size() const { return world_size_; }
  const std::vector<int>& devices() const { return devices_; }
  // Number of distinct devices the ranks use.
  int device_span() const;
  // The native single-process group (streams, peer access, partial buffers),
  // created on first multi-device use.
  tbik_local_group* native() const;

 private:
  int world_size_;
  std::vector<int> devices_;
  mutable std::shared_ptr<tbik_local_group> native_;
};

TBIK_CPP_API std::vector<Matrix> all_gather(const DeviceGroup& group, const std::vector<Matrix>& x_per_rank);

TBIK_CPP_API std::vector<Matrix> tree_all_reduce_per_rank(const DeviceGroup& group,
                                                          const std::vector<Matrix>& x_per_rank);

TBIK_CPP_API Matrix tree_all_reduce(const DeviceGroup& group, const std::vector<Matrix>& x_per_rank);

// Labelled non-invariant stand-in (left-to-right), a divergence baseline only.
TBIK_CPP_API Matrix ring_reduce_baseline(const DeviceGroup& group, const std::vector<Matrix>& x_per_rank);

}  // namespace tbik
