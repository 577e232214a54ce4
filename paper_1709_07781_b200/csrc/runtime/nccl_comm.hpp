// Internal: NCCL communicator of the multi-GPU build.
//
// libnccl is opened at run time (dlopen) the first time a communicator is
// made, so the runtime library has no link-time NCCL dependency and a
// process that never builds across GPUs never loads it.  When the process
// already has an NCCL loaded (e.g. PyTorch's), that one is used.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <string>

namespace ndactor::detail {

using NcclId = std::array<std::uint8_t, 128>;

class NcclComm {
 public:
  /// A fresh id for one communicator (rank 0 makes it, every rank gets a copy).
  static NcclId unique_id();

  /// Joins the communicator (collective over all ranks; this thread's
  /// current device must be the rank's GPU).
  NcclComm(int nranks, int rank, const NcclId& id);
  ~NcclComm();
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;

  int nranks() const { return nranks_; }
  int rank() const { return rank_; }

  /// recv = the ranks' `bytes` each, rank-major (ncclAllGather on uint8).
  /// Returns 0 or an NCCL error code; call between group_start/group_end to
  /// fuse several into one launch.
  int allgather(const void* send, void* recv, std::size_t bytes, void* stream) const;
  int group_start() const;
  int group_end() const;
  static std::string error_string(int rc);

 private:
  void* comm_ = nullptr;
  int nranks_ = 0, rank_ = 0;
};

}  // namespace ndactor::detail
