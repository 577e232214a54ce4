// extern "C" surface of the runtime (include/ndactor_c.h).
#include "ndactor_c.h"

#include <chrono>
#include <stdexcept>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <future>
#include <mutex>
#include <string>
#include <thread>

#include "ndactor/compute_actor.hpp"
#include "ndactor/wah_dist.hpp"
#include "nccl_comm.hpp"
#include "ndactor/wah_device.hpp"
#include "ndactor/wah_io.hpp"
#include "ndactor/wah_shard.hpp"
#include "ndx.h"

using namespace ndactor;

struct ndactor_runtime {
  std::unique_ptr<Device> dev;
  std::unique_ptr<ActorSystem> sys;
  wah::IndexStages stages;
  wah::IndexStages shard;  // stages for a nonzero row base (multi-GPU shards)
  std::uint32_t shard_base = 0;
  wah::DeviceIndex last;   // result of the last device build (kept alive)
  ActorHandle probe;
  // Pipelined host builds.  Three streams, so both PCIe directions and the
  // SMs work at once: uploads on `upload`, the build on the device stream,
  // the result copy on `egress` (the copy engines, no SMs).  The result size
  // is known only on the device: the build's last command copies the counts
  // to pinned memory and hands the slot to the egress thread, which issues
  // exactly W + 3D words of D2H once the counts have landed.
  struct Slot {
    Buffer keys;
    std::uint64_t cap = 0;
    void* uploaded = nullptr;  // cudaEvent: keys are on the device
    void* built = nullptr;     // cudaEvent: the counts are in `hc`
    void* done = nullptr;      // cudaEvent: the result is in host memory
    ndx_wah_counts* hc = nullptr;  // pinned
    MemRef cfg, words, entries;    // device result, held until the copy is done
    uint32_t* h_words = nullptr;
    uint32_t* h_entries = nullptr;
    std::uint64_t words_cap = 0, entries_cap = 0;
    ndx_wah_counts* counts = nullptr;
    bool busy = false;
    bool issued = false;  // egress has issued the copy (or failed)
    int rc = 0;
  };
  void* upload = nullptr;
  void* egress = nullptr;
  Slot slots[2];
  std::uint64_t next_ticket = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<int> jobs;
  bool stop = false;
  std::thread egress_thread;

  void egress_loop() {
    for (;;) {
      int j;
      {
        std::unique_lock<std::mutex> l(mu);
        cv.wait(l, [&] { return stop || !jobs.empty(); });
        if (jobs.empty()) return;
        j = jobs.front();
        jobs.pop_front();
      }
      Slot& sl = slots[j];
      int rc = ndx_event_synchronize(sl.built);
      if (!rc) {
        const ndx_wah_counts c = *sl.hc;
        *sl.counts = c;
        const std::uint64_t nw = std::min<std::uint64_t>(c.words, sl.words_cap);
        const std::uint64_t ne = std::min<std::uint64_t>(3 * c.distinct, sl.entries_cap);
        if (nw) rc = ndx_memcpy_d2h_async(sl.h_words, sl.words.buffer().data(), nw * 4, egress);
        if (!rc && ne) rc = ndx_memcpy_d2h_async(sl.h_entries, sl.entries.buffer().data(), ne * 4, egress);
        if (!rc) rc = ndx_event_record(sl.done, egress);
      }
      {
        std::lock_guard<std::mutex> l(mu);
        sl.issued = true;
        sl.rc = rc;
      }
      cv.notify_all();
    }
  }
  void post(int j, int rc) {
    {
      std::lock_guard<std::mutex> l(mu);
      if (rc) {
        slots[j].issued = true;
        slots[j].rc = rc;
      } else {
        jobs.push_back(j);
      }
    }
    cv.notify_all();
  }
  ~ndactor_runtime() {
    if (egress_thread.joinable()) {
      {
        std::lock_guard<std::mutex> l(mu);
        stop = true;
      }
      cv.notify_all();
      egress_thread.join();
    }
    if (egress) ndx_stream_synchronize(egress);  // copies issued but never waited for
    for (Slot& s : slots) {
      if (s.uploaded) ndx_event_destroy(s.uploaded);
      if (s.built) ndx_event_destroy(s.built);
      if (s.done) ndx_event_destroy(s.done);
      if (s.hc) ndx_host_free(s.hc);
    }
    if (upload) ndx_stream_destroy(upload);
    if (egress) ndx_stream_destroy(egress);
  }
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
  } catch (...) {
    g_err = "unknown error";
  }
  return -1;
}

}  // namespace

extern "C" {

const char* ndactor_last_error(void) { return g_err.c_str(); }

int ndactor_runtime_create(int device_ordinal, unsigned workers, ndactor_runtime** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null out pointer");
    auto rt = std::make_unique<ndactor_runtime>();
    DeviceConfig cfg;
    cfg.ordinal = device_ordinal;
    rt->dev = std::make_unique<Device>(cfg);
    rt->sys = std::make_unique<ActorSystem>(workers ? workers : 2u);
    rt->stages = wah::spawn_index_stages(*rt->sys, *rt->dev);
    *out = rt.release();
    return 0;
  });
}

void ndactor_runtime_destroy(ndactor_runtime* rt) {
  if (!rt) return;
  try {
    rt->last = wah::DeviceIndex{};
    rt->sys->await_idle();
    rt->dev->await_all();
    rt->sys->shutdown();
  } catch (...) {
  }
  delete rt;
}

void* ndactor_runtime_stream(ndactor_runtime* rt) { return rt ? rt->dev->stream() : nullptr; }

int ndactor_runtime_synchronize(ndactor_runtime* rt) {
  return guarded([&] {
    rt->dev->await_all();
    return 0;
  });
}

int ndactor_wah_build_index(ndactor_runtime* rt, const uint32_t* values, uint64_t n,
                            uint32_t row_base, uint32_t* words, uint64_t words_cap,
                            uint32_t* entries, uint64_t entries_cap, uint64_t* n_words,
                            uint64_t* n_entries) {
  return guarded([&] {
    if (!rt) throw std::invalid_argument("null runtime");
    if (n_words) *n_words = 0;
    if (n_entries) *n_entries = 0;
    if (n == 0) return 0;
    if (n >= (uint64_t(1) << 31)) throw std::length_error("a build takes at most 2^31 - 1 values");
    if (row_base != 0) throw std::invalid_argument("row_base needs ndactor_wah_build_index_device");
    Device& dev = *rt->dev;
    Buffer keys = dev.create_buffer_uninit(ElemType::u32, std::int64_t(n));
    Event wrote = dev.enqueue_native(
        "h2d_keys", [&](void* s) { return ndx_memcpy_h2d_async(keys.data(), values, n * 4, s); }, {});
    wah::DeviceIndex d = wah::build_index_device(*rt->sys, rt->stages, MemRef(keys, wrote), std::uint32_t(n));
    // counts, then exactly W words and D entries straight into the caller's buffers
    ndx_wah_counts c{};
    std::vector<Event> deps{d.entries.pending()};
    Event got = dev.enqueue_native(
        "d2h_counts", [&](void* s) { return ndx_memcpy_d2h_async(&c, d.cfg.buffer().data(), sizeof c, s); },
        deps);
    if (got.await() == EventState::failed) throw std::runtime_error(got.error());
    if (c.words > words_cap || 3 * c.distinct > entries_cap) throw std::length_error("output buffers too small");
    Event rd = dev.enqueue_native(
        "d2h_index",
        [&](void* s) -> int {
          int rc = ndx_memcpy_d2h_async(words, d.words.buffer().data(), c.words * 4, s);
          if (!rc) rc = ndx_memcpy_d2h_async(entries, d.entries.buffer().data(), c.distinct * 12, s);
          return rc;
        },
        {});
    if (rd.await() == EventState::failed) throw std::runtime_error(rd.error());
    release(d.cfg);
    release(d.words);
    release(d.entries);
    if (n_words) *n_words = c.words;
    if (n_entries) *n_entries = c.distinct;
    return 0;
  });
}

int ndactor_wah_build_index_async(ndactor_runtime* rt, const uint32_t* values, uint64_t n,
                                  uint32_t* words, uint64_t words_cap, uint32_t* entries,
                                  uint64_t entries_cap, ndx_wah_counts* counts, uint64_t* ticket) {
  return guarded([&] {
    if (!rt || !counts || !ticket) throw std::invalid_argument("null argument");
    if (n == 0) throw std::invalid_argument("empty input");
    if (n >= (uint64_t(1) << 31)) throw std::length_error("a build takes at most 2^31 - 1 values");
    if ((!words && words_cap) || (!entries && entries_cap)) throw std::invalid_argument("null output buffer");
    Device& dev = *rt->dev;
    auto ck = [](int rc, const char* what) {
      if (rc) throw std::runtime_error(std::string(what) + ": " + ndx_error_string(rc));
    };
    if (!rt->upload) ck(ndx_stream_create(&rt->upload), "upload stream");
    if (!rt->egress) ck(ndx_stream_create(&rt->egress), "egress stream");
    if (!rt->egress_thread.joinable()) rt->egress_thread = std::thread([rt] { rt->egress_loop(); });
    const std::uint64_t t = rt->next_ticket;
    const int j = int(t & 1);
    ndactor_runtime::Slot& sl = rt->slots[j];
    if (sl.busy) throw std::runtime_error("two builds already in flight: wait for one first");
    if (!sl.uploaded) ck(ndx_event_create(&sl.uploaded, 0), "event");
    if (!sl.built) ck(ndx_event_create(&sl.built, 0), "event");
    if (!sl.done) ck(ndx_event_create(&sl.done, 0), "event");
    if (!sl.hc) ck(ndx_host_alloc(reinterpret_cast<void**>(&sl.hc), sizeof(ndx_wah_counts)), "pinned counts");
    if (sl.cap < n) {
      if (sl.keys.valid()) {
        dev.await_all();
        dev.free_buffer(sl.keys);
      }
      sl.keys = dev.create_buffer_uninit(ElemType::u32, std::int64_t(n));
      sl.cap = n;
      dev.await_all();
    }
    // the slot's keys were last read by build t-2, whose result copy (`done`)
    // came after it
    ck(ndx_stream_wait_event(rt->upload, sl.done), "upload wait");
    ck(ndx_memcpy_h2d_async(sl.keys.data(), values, n * 4, rt->upload), "upload");
    ck(ndx_event_record(sl.uploaded, rt->upload), "upload record");
    void* up = sl.uploaded;
    Event ready = dev.enqueue_native("wait_upload", [up](void* s) { return ndx_stream_wait_event(s, up); }, {});
    // the chain releases its input MemRef: hand it a non-owning view of the slot
    Buffer view = dev.wrap_buffer(sl.keys.data(), ElemType::u32, std::int64_t(n), Access::read_only);
    wah::DeviceIndex d = wah::build_index_device(*rt->sys, rt->stages, MemRef(view, ready), std::uint32_t(n));
    sl.cfg = d.cfg;
    sl.words = d.words;
    sl.entries = d.entries;
    sl.h_words = words;
    sl.h_entries = entries;
    sl.words_cap = words_cap;
    sl.entries_cap = entries_cap;
    sl.counts = counts;
    sl.issued = false;
    sl.rc = 0;
    std::vector<Event> deps{d.entries.pending(), d.words.pending(), d.cfg.pending()};
    const void* cfg = d.cfg.buffer().data();
    ndx_wah_counts* hc = sl.hc;
    void* built = sl.built;
    Event counted = dev.enqueue_native(
        "counts_d2h",
        [=](void* s) -> int {
          int rc = ndx_memcpy_d2h_async(hc, cfg, sizeof(ndx_wah_counts), s);
          if (!rc) rc = ndx_event_record(built, s);
          rt->post(j, rc);
          return rc;
        },
        deps);
    // a command that never runs (device failure upstream) still ends the wait
    counted.add_callback([rt, j](EventState st) {
      if (st == EventState::failed) rt->post(j, -1);
    });
    sl.busy = true;
    rt->next_ticket = t + 1;
    *ticket = t;
    return 0;
  });
}

int ndactor_wah_wait(ndactor_runtime* rt, uint64_t ticket) {
  return guarded([&] {
    if (!rt) throw std::invalid_argument("null runtime");
    ndactor_runtime::Slot& sl = rt->slots[ticket & 1];
    if (!sl.busy) return 0;
    (void)rt->dev->stream();  // every queued launch issued
    int rc;
    {
      std::unique_lock<std::mutex> l(rt->mu);
      rt->cv.wait(l, [&] { return sl.issued; });
      rc = sl.rc;
    }
    if (!rc) rc = ndx_event_synchronize(sl.done);
    release(sl.cfg);
    release(sl.words);
    release(sl.entries);
    sl.cfg = sl.words = sl.entries = MemRef{};
    sl.busy = false;
    if (rc) throw std::runtime_error(std::string("build failed: ") + (rc > 0 ? ndx_error_string(rc) : "device failure"));
    return 0;
  });
}

int ndactor_wah_build_index_device(ndactor_runtime* rt, const uint32_t* d_keys, uint64_t n,
                                   uint32_t row_base, uint32_t** d_words, uint32_t** d_entries,
                                   void** d_counts) {
  return guarded([&] {
    if (!rt) throw std::invalid_argument("null runtime");
    rt->last = wah::DeviceIndex{};  // previous result: released in stream order
    if (n == 0) return 0;
    if (n >= (uint64_t(1) << 31)) throw std::length_error("a build takes at most 2^31 - 1 values");
    if (uint64_t(row_base) + n > (uint64_t(1) << 32))
      throw std::length_error("row ids row_base .. row_base + n - 1 must fit in u32");
    Device& dev = *rt->dev;
    wah::IndexStages* st = &rt->stages;
    if (row_base != 0) {
      if (!rt->shard.chain.valid() || rt->shard_base != row_base) {
        if (rt->shard.chain.valid())
          for (const ActorHandle& a : {rt->shard.chain, rt->shard.table, rt->shard.emit, rt->shard.sort,
                                       rt->shard.plan})
            rt->sys->terminate(a);
        rt->shard = wah::spawn_index_stages(*rt->sys, dev, row_base);
        rt->shard_base = row_base;
      }
      st = &rt->shard;
    }
    Buffer keys = dev.wrap_buffer(const_cast<uint32_t*>(d_keys), ElemType::u32, std::int64_t(n),
                                  Access::read_only);
    rt->last = wah::build_index_device(*rt->sys, *st, MemRef(keys, Event{}), std::uint32_t(n));
    if (d_words) *d_words = static_cast<uint32_t*>(rt->last.words.buffer().data());
    if (d_entries) *d_entries = static_cast<uint32_t*>(rt->last.entries.buffer().data());
    if (d_counts) *d_counts = rt->last.cfg.buffer().data();
    return 0;
  });
}

namespace {

// Chain `iters` requests through `actor`, each issued from the previous
// reply; returns the last reply.
Reply chain_requests(ActorSystem& sys, ActorHandle actor, Message first, uint64_t iters) {
  struct Loop {
    ActorSystem* sys;
    ActorHandle actor;
    uint64_t left;
    std::promise<Reply> done;
    std::function<void(Reply)> step;
  };
  auto loop = std::make_shared<Loop>();
  loop->sys = &sys;
  loop->actor = actor;
  loop->left = iters;
  Loop* lp = loop.get();
  loop->step = [lp](Reply r) {
    if (is_error(r) || --lp->left == 0) {
      lp->done.set_value(std::move(r));
      return;
    }
    lp->sys->request(lp->actor, std::move(std::get<Message>(r))).then(std::ref(lp->step));
  };
  auto fut = loop->done.get_future();
  sys.request(actor, std::move(first)).then(std::ref(loop->step));
  Reply last = fut.get();
  sys.await_idle();
  return last;
}

ActorHandle tiny_actor(ActorSystem& sys, Device& dev, bool launch) {
  ComputeActorSpec spec;
  if (launch)
    spec.kernel = KernelDef("tiny_increment", [](const LaunchParams& lp) -> int {
      return ndx_tiny_increment(static_cast<uint32_t*>(lp.ptr[0]), lp.stream);
    });
  else
    spec.kernel = KernelDef("host_only", [](const LaunchParams&) -> int { return 0; });
  spec.range = NdRange::linear(32, 32);
  spec.args = {ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref)};
  return spawn_compute(sys, dev, std::move(spec));
}

}  // namespace

int ndactor_dispatch_probe_ex(ndactor_runtime* rt, uint64_t iters, double* out /* [5] */) {
  return guarded([&] {
    Device& dev = *rt->dev;
    ActorSystem& sys = *rt->sys;
    using clk = std::chrono::steady_clock;
    auto ms_since = [](clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); };
    Buffer counter = dev.create_buffer(ElemType::u32, 1);
    dev.await_all();

    // (a) raw: back-to-back launches on the runtime stream, one sync
    void* stream = dev.stream();
    auto t0 = clk::now();
    for (uint64_t i = 0; i < iters; ++i) {
      int rc = ndx_tiny_increment(static_cast<uint32_t*>(counter.data()), stream);
      if (rc) throw std::runtime_error(ndx_error_string(rc));
    }
    out[1] = ms_since(t0);  // host enqueue time alone
    ndx_stream_synchronize(dev.stream());
    out[0] = ms_since(t0);

    // (b) through a compute actor, each request issued from the previous reply
    if (!rt->probe.valid()) rt->probe = tiny_actor(sys, dev, true);
    MemRef ref(counter, Event{});
    auto t1 = clk::now();
    Reply last = chain_requests(sys, rt->probe, Message::of(ref), iters);
    if (is_error(last)) throw std::runtime_error(get_error(last).what);
    std::vector<uint32_t> v = retrieve_u32(get_message(last).at(0).as_ref());
    out[2] = ms_since(t1);
    out[4] = v.empty() ? 0 : double(v[0]);

    // (c) the same chain with a launcher that issues nothing: host cost of a hop
    ActorHandle host_only = tiny_actor(sys, dev, false);
    auto t2 = clk::now();
    Reply l2 = chain_requests(sys, host_only, Message::of(get_message(last).at(0).as_ref()), iters);
    out[3] = ms_since(t2);
    sys.terminate(host_only);
    return 0;
  });
}

int ndactor_dispatch_probe(ndactor_runtime* rt, uint64_t iters, double* raw_ms, double* actor_ms,
                           uint64_t* check) {
  double r[5] = {};
  int rc = ndactor_dispatch_probe_ex(rt, iters, r);
  if (rc) return rc;
  *raw_ms = r[0];
  *actor_ms = r[2];
  if (check) *check = uint64_t(r[4]);
  return 0;
}

int ndactor_write_index_file(const char* path, uint32_t row_count, const uint32_t* entries,
                             uint64_t n_entries, const uint32_t* words, uint64_t n_words) {
  return guarded([&] {
    wah::WahIndex idx;
    idx.row_count = row_count;
    idx.entries.resize(n_entries);
    for (uint64_t i = 0; i < n_entries; ++i)
      idx.entries[i] = wah::IndexEntry{entries[3 * i], entries[3 * i + 1], entries[3 * i + 2]};
    idx.words.assign(words, words + n_words);
    wah::write_index_file(path, idx);
    return 0;
  });
}

// FNV-1a-64 over the "WAH1" serialization, streamed from the parts (no
// serialized copy): the digest the parity fixtures and SURVEY App. C use.
uint64_t ndactor_index_digest(uint32_t row_count, const uint32_t* entries, uint64_t n_entries,
                              const uint32_t* words, uint64_t n_words) {
  uint64_t h = 1469598103934665603ull;
  auto bytes = [&h](const void* p, uint64_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (uint64_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  auto u32 = [&bytes](uint32_t v) {
    const unsigned char le[4] = {uint8_t(v), uint8_t(v >> 8), uint8_t(v >> 16), uint8_t(v >> 24)};
    bytes(le, 4);
  };
  bytes("WAH1", 4);
  u32(row_count);
  u32(uint32_t(n_entries));
  u32(uint32_t(n_words));
  if (n_entries) bytes(entries, 12 * n_entries);  // little-endian host
  if (n_words) bytes(words, 4 * n_words);
  return h;
}

// ---- multi-GPU build (include/ndactor/wah_dist.hpp) ------------------------

struct ndactor_dist {
  ndactor_runtime* rt;
  std::unique_ptr<wah::DistBuild> build;
};

int ndactor_nccl_unique_id(uint8_t* id128) {
  return guarded([&] {
    if (!id128) throw std::invalid_argument("null id buffer");
    const detail::NcclId id = detail::NcclComm::unique_id();
    std::memcpy(id128, id.data(), id.size());
    return 0;
  });
}

int ndactor_dist_create(ndactor_runtime* rt, int rank, int nranks, const uint8_t* id128, uint64_t local_cap,
                        uint32_t meta_cap, uint64_t slice_cap, ndactor_dist** out) {
  return guarded([&] {
    if (!rt || !id128 || !out) throw std::invalid_argument("null argument");
    detail::NcclId id;
    std::memcpy(id.data(), id128, id.size());
    auto d = std::make_unique<ndactor_dist>();
    d->rt = rt;
    d->build = std::make_unique<wah::DistBuild>(*rt->sys, *rt->dev, rank, nranks, id, local_cap, meta_cap, slice_cap);
    *out = d.release();
    return 0;
  });
}

int ndactor_dist_step(ndactor_dist* d, const uint32_t* d_keys, uint64_t n_local, uint64_t row_base, int gather_all) {
  return guarded([&] {
    if (!d || !d_keys) throw std::invalid_argument("null argument");
    d->build->step(d_keys, n_local, row_base, gather_all != 0);
    return 0;
  });
}

int ndactor_dist_outputs(ndactor_dist* d, uint64_t** d_totals, uint64_t** d_bounds, uint32_t** d_entries,
                         uint32_t** d_slice, uint32_t** d_local_words) {
  return guarded([&] {
    if (!d) throw std::invalid_argument("null argument");
    if (d_totals) *d_totals = const_cast<uint64_t*>(d->build->totals());
    if (d_bounds) *d_bounds = const_cast<uint64_t*>(d->build->bounds());
    if (d_entries) *d_entries = const_cast<uint32_t*>(d->build->entries());
    if (d_slice) *d_slice = const_cast<uint32_t*>(d->build->slice());
    if (d_local_words) *d_local_words = const_cast<uint32_t*>(d->build->local_words());
    return 0;
  });
}

void ndactor_dist_destroy(ndactor_dist* d) {
  try {
    delete d;
  } catch (...) {
  }
}

int ndactor_shard_bounds(uint64_t n, uint32_t shards, uint64_t* bounds) {
  return guarded([&] {
    const auto b = wah::shard_bounds(n, shards);
    std::memcpy(bounds, b.data(), b.size() * sizeof(uint64_t));
    return 0;
  });
}

int ndactor_merge_plan(uint32_t shards, const ndx_shard_meta* metas, const uint64_t* counts,
                       uint64_t stride, uint32_t* entries, ndx_piece* pieces, uint64_t* n_entries,
                       uint64_t* n_words) {
  return guarded([&] {
    static_assert(sizeof(wah::IndexEntry) == 12, "IndexEntry must be three u32");
    std::vector<std::span<const ndx_shard_meta>> sh(shards);
    std::vector<ndx_piece*> outs(shards);
    std::uint64_t off = 0;
    for (uint32_t g = 0; g < shards; ++g) {
      const std::uint64_t at = stride ? g * stride : off;
      sh[g] = std::span<const ndx_shard_meta>(metas + at, counts[g]);
      outs[g] = pieces + at;
      off += counts[g];
    }
    auto [ne, nw] = wah::plan_merge_into(sh, reinterpret_cast<wah::IndexEntry*>(entries), outs);
    *n_entries = ne;
    *n_words = nw;
    return 0;
  });
}

}  // extern "C"
