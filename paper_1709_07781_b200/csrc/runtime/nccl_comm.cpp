// NCCL through dlopen: the handful of entry points the multi-GPU build uses.
#include "nccl_comm.hpp"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <stdexcept>

namespace ndactor::detail {

namespace {

struct UniqueId {
  char internal[128];
};

struct Nccl {
  int (*get_unique_id)(UniqueId*) = nullptr;
  int (*comm_init_rank)(void**, int, UniqueId, int) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*all_gather)(const void*, void*, std::size_t, int, void*, void*) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  const char* (*error_string)(int) = nullptr;
  std::string why;  // empty: loaded
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("cannot load libnccl: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && n.why.empty()) n.why = std::string("libnccl lacks ") + name;
      return p;
    };
    n.get_unique_id = reinterpret_cast<int (*)(UniqueId*)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<int (*)(void**, int, UniqueId, int)>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<int (*)(void*)>(sym("ncclCommDestroy"));
    n.all_gather =
        reinterpret_cast<int (*)(const void*, void*, std::size_t, int, void*, void*)>(sym("ncclAllGather"));
    n.group_start = reinterpret_cast<int (*)()>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<int (*)()>(sym("ncclGroupEnd"));
    n.error_string = reinterpret_cast<const char* (*)(int)>(sym("ncclGetErrorString"));
  });
  if (!n.why.empty()) throw std::runtime_error(n.why);
  return n;
}

constexpr int kNcclUint8 = 1;  // ncclDataType_t

void check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string(what) + ": " + NcclComm::error_string(rc));
}

}  // namespace

NcclId NcclComm::unique_id() {
  UniqueId u{};
  check(nccl().get_unique_id(&u), "ncclGetUniqueId");
  NcclId id{};
  std::memcpy(id.data(), u.internal, id.size());
  return id;
}

NcclComm::NcclComm(int nranks, int rank, const NcclId& id) : nranks_(nranks), rank_(rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad NCCL rank / size");
  UniqueId u{};
  std::memcpy(u.internal, id.data(), id.size());
  check(nccl().comm_init_rank(&comm_, nranks, u, rank), "ncclCommInitRank");
}

NcclComm::~NcclComm() {
  if (comm_) nccl().comm_destroy(comm_);
}

int NcclComm::allgather(const void* send, void* recv, std::size_t bytes, void* stream) const {
  return nccl().all_gather(send, recv, bytes, kNcclUint8, comm_, stream);
}
int NcclComm::group_start() const { return nccl().group_start(); }
int NcclComm::group_end() const { return nccl().group_end(); }

std::string NcclComm::error_string(int rc) {
  try {
    const Nccl& n = nccl();
    if (n.error_string) return n.error_string(rc);
  } catch (...) {
  }
  return "NCCL error " + std::to_string(rc);
}

}  // namespace ndactor::detail
