// ndactor/wah_dist.hpp -- the multi-GPU WAH build behind the actor API
// (the paper's stated future work).
//
// One DistBuild per rank (one process per GPU).  Each step builds the rank's
// row shard through the shard chain (compute actors, global row ids), then --
// stream-ordered on the rank's device, no host round trip -- all-gathers
// every shard's counts and per-value metadata over NCCL, plans the boundary
// merge (Appendix B) on the GPU, and copies the rank's owned slice of the
// merged words (or, gather_all, all of them) straight out of the other GPUs'
// word buffers over NVLink.  The merged table is replicated on every rank.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "ndactor/wah_device.hpp"

namespace ndactor::detail {
class NcclComm;  // the runtime's NCCL binding (libnccl opened at run time)
using NcclId = std::array<std::uint8_t, 128>;
}  // namespace ndactor::detail

namespace ndactor::wah {

class DistBuild {
 public:
  /// local_cap: the largest shard (values); meta_cap: the most distinct
  /// values a shard may hold (the metadata all-gather is sized by it; a
  /// shard with more is flagged in the step's error word); slice_cap: the
  /// words the rank's output holds.
  DistBuild(ActorSystem& sys, Device& dev, int rank, int nranks, const detail::NcclId& id,
            std::uint64_t local_cap, std::uint32_t meta_cap, std::uint64_t slice_cap);
  ~DistBuild();
  DistBuild(const DistBuild&) = delete;
  DistBuild& operator=(const DistBuild&) = delete;

  /// Enqueues one step over this rank's n keys (device memory) with row ids
  /// row_base .. row_base + n - 1; returns without waiting.
  void step(const std::uint32_t* d_keys, std::uint64_t n, std::uint64_t row_base, bool gather_all);

  /// Device outputs of the last step (valid once the device stream is past it):
  /// totals {D, W, error flags, records}, bounds[0..G] (owned words of rank h:
  /// [bounds[h], bounds[h+1])), the merged (value, offset, length) table, the
  /// slice (the owned words, or all of them after a gather step).
  const std::uint64_t* totals() const { return static_cast<const std::uint64_t*>(totals_.data()); }
  const std::uint64_t* bounds() const { return static_cast<const std::uint64_t*>(bounds_.data()); }
  const std::uint32_t* entries() const { return static_cast<const std::uint32_t*>(entries_.data()); }
  const std::uint32_t* slice() const {
    return single_ ? local_words() : static_cast<const std::uint32_t*>(slice_.data());
  }
  /// The rank's own shard words of the last step (its local index).
  const std::uint32_t* local_words() const { return static_cast<const std::uint32_t*>(wbuf_[parity_ ^ 1]); }

 private:
  struct Step {
    MemRef cfg, words, entries, meta;
    Event done;
  };
  ActorSystem& sys_;
  Device& dev_;
  int rank_, nranks_;
  std::uint64_t local_cap_;
  std::uint32_t meta_cap_;
  std::uint64_t slice_cap_;
  std::unique_ptr<detail::NcclComm> comm_;
  ShardStages stages_;
  std::uint64_t stages_base_ = ~std::uint64_t(0);
  void* wbuf_[2] = {nullptr, nullptr};
  std::vector<const std::uint32_t*> peers_[2];
  std::vector<void*> opened_;
  Buffer metas_all_, counts_all_, entries_, merged_, totals_, bounds_, scratch_, slice_;
  Step keep_;
  int parity_ = 0;
  bool single_ = false;  // one shard: the slice is the local words
};

}  // namespace ndactor::wah
