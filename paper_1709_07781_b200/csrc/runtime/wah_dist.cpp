// Multi-GPU WAH build: one process per GPU, one step per call, every stage
// stream-ordered on the rank's device with no host round trip
// (SURVEY.md section 8(e), Appendix B).
//
//   1. the local build of the rank's row shard through the shard chain
//      (plan * sort * emit * table * meta; global row ids; the words in a
//      buffer the other GPUs have mapped over NVLink)
//   2. one NCCL group: all-gather of every shard's counts and metadata
//   3. the merge plan, replicated on every rank (ndx_dist_plan): the merged
//      table, the pieces in destination order, the owner bounds
//   4. the exchange as one kernel (ndx_dist_pull): each rank copies the
//      pieces of its owned value range -- or rank 0 everything (gather) --
//      straight out of the other GPUs' word buffers
//
// The word buffers alternate between steps: a rank may rewrite buffer p only
// after every rank has passed the next step's all-gather, which every rank
// issues after its pull of the step before.
#include "ndactor/wah_dist.hpp"

#include <cstring>
#include <stdexcept>

#include "device_impl.hpp"
#include "nccl_comm.hpp"
#include "ndx.h"

namespace ndactor::wah {

namespace {
void ck(int rc, const char* what) {
  if (rc != 0) throw DeviceError(std::string(what) + ": " + ndx_error_string(rc));
}
}  // namespace

DistBuild::DistBuild(ActorSystem& sys, Device& dev, int rank, int nranks, const detail::NcclId& id,
                     std::uint64_t local_cap, std::uint32_t meta_cap, std::uint64_t slice_cap)
    : sys_(sys), dev_(dev), rank_(rank), nranks_(nranks), local_cap_(local_cap), meta_cap_(meta_cap),
      slice_cap_(slice_cap) {
  if (nranks < 1 || nranks > 64) throw std::invalid_argument("1 to 64 ranks");
  if (local_cap == 0 || meta_cap == 0) throw std::invalid_argument("empty capacities");
  ck(detail::bind_thread(dev.impl().ordinal), "bind device");
  comm_ = std::make_unique<detail::NcclComm>(nranks, rank, id);
  const std::uint64_t G = std::uint64_t(nranks);
  const std::uint64_t rec = G * meta_cap;
  for (int p = 0; p < 2; ++p) ck(ndx_malloc_shared(&wbuf_[p], 2 * local_cap * 4), "word buffer");
  metas_all_ = dev.create_buffer_uninit(ElemType::u32, std::int64_t(rec * (sizeof(ndx_shard_meta) / 4)));
  counts_all_ = dev.create_buffer_uninit(ElemType::u32, std::int64_t(G * (sizeof(ndx_wah_counts) / 4)));
  entries_ = dev.create_buffer_uninit(ElemType::u32, std::int64_t(3 * rec + 3));
  merged_ = dev.create_buffer_uninit(ElemType::u32, std::int64_t((rec + 1) * (sizeof(ndx_piece) / 4)));
  totals_ = dev.create_buffer(ElemType::u32, 2 * 4);
  bounds_ = dev.create_buffer(ElemType::u32, std::int64_t(2 * (G + 1)));
  scratch_ = dev.create_buffer_uninit(ElemType::u32,
                                      std::int64_t(ndx_dist_plan_scratch_bytes(std::uint32_t(G), meta_cap) / 4 + 64));
  slice_ = dev.create_buffer_uninit(ElemType::u32, std::int64_t(slice_cap + 1));

  // every rank maps every other rank's word buffers (CUDA IPC), the handles
  // travel by one all-gather
  for (int p = 0; p < 2; ++p) peers_[p].assign(G, nullptr);
  if (G > 1) {
    std::vector<std::uint8_t> mine(128), all(128 * G);
    ck(ndx_ipc_handle(wbuf_[0], mine.data()), "IPC handle");
    ck(ndx_ipc_handle(wbuf_[1], mine.data() + 64), "IPC handle");
    Buffer hb = dev.create_buffer_uninit(ElemType::u32, 32);
    Buffer ha = dev.create_buffer_uninit(ElemType::u32, std::int64_t(32 * G));
    Event ex = dev.enqueue_native(
        "exchange_ipc_handles",
        [&](void* s) -> int {
          int rc = ndx_memcpy_h2d_async(hb.data(), mine.data(), 128, s);
          if (rc) return rc;
          if ((rc = comm_->allgather(hb.data(), ha.data(), 128, s))) return NDX_E_INVALID;
          return ndx_memcpy_d2h_async(all.data(), ha.data(), 128 * G, s);
        },
        {});
    if (ex.await() == EventState::failed) throw DeviceError("IPC handle exchange: " + ex.error());
    dev.free_buffer(hb);
    dev.free_buffer(ha);
    for (std::uint64_t g = 0; g < G; ++g)
      for (int p = 0; p < 2; ++p) {
        if (int(g) == rank) continue;
        void* q = nullptr;
        ck(ndx_ipc_open(all.data() + 128 * g + 64 * p, &q), "IPC open");
        peers_[p][g] = static_cast<const std::uint32_t*>(q);
        opened_.push_back(q);
      }
  }
  for (int p = 0; p < 2; ++p) peers_[p][rank] = static_cast<const std::uint32_t*>(wbuf_[p]);
}

DistBuild::~DistBuild() {
  try {
    dev_.await_all();
  } catch (...) {
  }
  keep_ = {};
  if (stages_.chain.valid())
    for (const ActorHandle& a : {stages_.chain, stages_.meta, stages_.table, stages_.emit, stages_.sort, stages_.plan})
      sys_.terminate(a);
  for (void* q : opened_) ndx_ipc_close(q);
  for (Buffer* b : {&metas_all_, &counts_all_, &entries_, &merged_, &totals_, &bounds_, &scratch_, &slice_}) {
    try {
      if (b->valid()) dev_.free_buffer(*b);
    } catch (...) {
    }
  }
  try {
    dev_.await_all();
  } catch (...) {
  }
  for (void* w : wbuf_)
    if (w) ndx_free_shared(w);
  comm_.reset();
}

void DistBuild::step(const std::uint32_t* d_keys, std::uint64_t n, std::uint64_t row_base, bool gather_all) {
  if (n == 0 || n > local_cap_) throw std::length_error("shard size outside the build's capacity");
  if (row_base + n > (std::uint64_t(1) << 32)) throw std::length_error("row ids must fit in u32");
  if (!stages_.chain.valid() || stages_base_ != row_base) {
    if (stages_.chain.valid())
      for (const ActorHandle& a : {stages_.chain, stages_.meta, stages_.table, stages_.emit, stages_.sort, stages_.plan})
        sys_.terminate(a);
    stages_ = spawn_shard_stages(sys_, dev_, std::uint32_t(row_base), meta_cap_);
    stages_base_ = row_base;
  }
  const int p = parity_;
  parity_ ^= 1;
  MemRef keys(dev_.wrap_buffer(const_cast<std::uint32_t*>(d_keys), ElemType::u32, std::int64_t(n),
                               Access::read_only),
              Event{});
  MemRef words(dev_.wrap_buffer(wbuf_[p], ElemType::u32, std::int64_t(2 * local_cap_)), Event{});
  Reply r = sys_.request(stages_.chain, Message::of(std::move(keys), std::move(words))).await();
  if (is_error(r)) throw DeviceError("shard build failed: " + get_error(r).what);
  const Message& m = get_message(r);
  Step st;
  st.cfg = m.at(0).as_ref();
  st.words = m.at(1).as_ref();
  st.entries = m.at(2).as_ref();
  st.meta = m.at(3).as_ref();

  const std::uint32_t G = std::uint32_t(nranks_);
  void* counts_all = counts_all_.data();
  void* metas_all = metas_all_.data();
  const void* cfg = st.cfg.buffer().data();
  const void* meta = st.meta.buffer().data();
  const std::size_t meta_bytes = std::size_t(meta_cap_) * sizeof(ndx_shard_meta);
  detail::NcclComm* comm = comm_.get();
  std::vector<Event> after{st.meta.pending()};
  Event ag = dev_.enqueue_native(
      "meta_allgather",
      [=](void* s) -> int {
        if (comm->group_start()) return NDX_E_INVALID;
        const int a = comm->allgather(cfg, counts_all, sizeof(ndx_wah_counts), s);
        const int b = comm->allgather(meta, metas_all, meta_bytes, s);
        const int c = comm->group_end();
        return (a || b || c) ? NDX_E_INVALID : 0;
      },
      after);
  ndx_piece* merged = static_cast<ndx_piece*>(merged_.data());
  std::uint64_t* totals = static_cast<std::uint64_t*>(totals_.data());
  std::uint64_t* bounds = static_cast<std::uint64_t*>(bounds_.data());
  std::uint32_t* entries = static_cast<std::uint32_t*>(entries_.data());
  void* scratch = scratch_.data();
  const std::uint32_t cap = meta_cap_;
  Event pl = dev_.enqueue_native(
      "merge_plan",
      [=](void* s) {
        return ndx_dist_plan(static_cast<const ndx_shard_meta*>(metas_all), cap,
                             static_cast<const ndx_wah_counts*>(counts_all), G, entries, merged, totals, bounds,
                             scratch, s);
      },
      {});
  // one shard: the plan maps every local word onto itself, the slice is the
  // local index as it stands (no copy)
  single_ = G == 1;
  if (single_) {
    keep_ = std::move(st);
    return;
  }
  const std::uint32_t* const* peers = peers_[p].data();
  std::uint32_t* slice = static_cast<std::uint32_t*>(slice_.data());
  const std::uint64_t slice_cap = slice_cap_;
  const std::uint64_t hint = gather_all ? 2 * n * G : 2 * n;
  const std::uint32_t rank = std::uint32_t(rank_);
  Event pu = dev_.enqueue_native(
      "pull_words",
      [=](void* s) {
        return ndx_dist_pull(peers, G, merged, std::uint64_t(G) * cap, totals, bounds, rank, gather_all ? 1 : 0,
                             slice, slice_cap, hint, s);
      },
      {});
  st.done = pu;
  keep_ = std::move(st);  // the step before: released here, freed in stream order
}

}  // namespace ndactor::wah
