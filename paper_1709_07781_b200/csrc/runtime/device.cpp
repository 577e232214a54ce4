// Device: CUDA stream + stream-ordered pool + completion thread.
// Replaces the reference's simulated device (p/core/src/device.cpp:45-348):
//   - command DAG of dependency callbacks  -> stream order (same device),
//     cudaStreamWaitEvent (other device), deferred issue (host events)
//   - worker threads executing work groups -> the GPU
//   - Event transitions                    -> a completion thread that
//     records one CUDA event only when somebody waits, and completes every
//     waiting event up to that stream position
#include "ndactor/device.hpp"

#include <algorithm>
#include <cstring>

#include "device_impl.hpp"
#include "ndx.h"

namespace ndactor {

namespace detail {

namespace {
std::string cuda_msg(int rc) { return ndx_error_string(rc); }
}  // namespace

// CUDA's current device is per host thread: every thread that touches this
// Device's stream, events or kernels binds to its ordinal first (cached, so
// the hot path pays one compare).
int bind_thread(int ordinal) {
  thread_local int bound = -1;
  if (bound == ordinal) return 0;
  const int rc = ndx_device_bind(ordinal);
  if (rc == 0) bound = ordinal;
  return rc;
}

void DeviceImpl::start() {
  completer = std::thread([this] {
    bind_thread(ordinal);
    completer_loop();
  });
  launcher = std::thread([this] {
    bind_thread(ordinal);
    launcher_loop();
  });
}

void DeviceImpl::stop() {
  {
    std::lock_guard<std::mutex> l(watch_mu);
    stopping = true;
  }
  watch_cv.notify_all();
  if (completer.joinable()) completer.join();
  {
    std::lock_guard<std::mutex> l(q_mu);
    q_stop = true;
  }
  q_cv.notify_all();
  if (launcher.joinable()) launcher.join();
}

namespace {
inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
  __builtin_ia32_pause();
#endif
}
}  // namespace

void DeviceImpl::push_launch(const LaunchParams& p, const Launcher& launch,
                             const std::shared_ptr<Event::State>& ev, std::uint64_t seq,
                             const std::string& name) {
  const std::uint64_t t = q_pushed.load(std::memory_order_relaxed);
  for (unsigned i = 0; t - q_done.load(std::memory_order_acquire) >= kRing; ++i)
    if (i > 64) std::this_thread::yield();  // ring full: the launcher is behind
  LaunchJob& j = ring[t % kRing];
  j.seq = seq;
  j.ev = ev;
  j.launch = launch;
  j.grid = p.grid;
  j.block = p.block;
  j.rank = p.rank;
  j.nargs = unsigned(p.nargs);
  j.shared_bytes = p.shared_bytes;
  j.offset = p.offset;
  j.global = p.global;
  if (p.nargs > kInlineArgs) j.more.reset(new LaunchArg[p.nargs - kInlineArgs]);
  for (std::size_t i = 0; i < p.nargs; ++i) {
    LaunchArg& a = i < kInlineArgs ? j.args[i] : j.more[i - kInlineArgs];
    a.ptr = p.ptr[i];
    a.len = p.len[i];
    a.smem_offset = p.smem_offset[i];
    a.scalar = p.scalar[i];
  }
  j.name_copy = name;
  // seq_cst pair with the launcher's (store sleeping, load pushed): one of
  // the two sides always sees the other
  q_pushed.store(t + 1, std::memory_order_seq_cst);
  if (q_sleeping.load(std::memory_order_seq_cst)) {
    std::lock_guard<std::mutex> l(q_mu);
    q_cv.notify_one();
  }
}

void DeviceImpl::drain() {
  const std::uint64_t target = q_pushed.load(std::memory_order_acquire);
  for (unsigned i = 0; q_done.load(std::memory_order_acquire) < target; ++i) {
    if (i < 4096)
      cpu_relax();
    else
      std::this_thread::yield();
  }
}

void DeviceImpl::launcher_loop() {
  std::uint64_t h = 0;
  LaunchParams lp;  // this thread's own copy, hot in its cache
  for (;;) {
    std::uint64_t t = q_pushed.load(std::memory_order_acquire);
    if (h == t) {
      // a chain of requests arrives every microsecond or so: spin briefly
      // before sleeping so a steady stream never pays a wake-up
      for (int i = 0; i < 20000 && (t = q_pushed.load(std::memory_order_acquire)) == h; ++i) cpu_relax();
      if (h == t) {
        std::unique_lock<std::mutex> l(q_mu);
        q_sleeping.store(true, std::memory_order_seq_cst);
        q_cv.wait(l, [&] { return q_stop || q_pushed.load(std::memory_order_seq_cst) != h; });
        q_sleeping.store(false, std::memory_order_release);
        t = q_pushed.load(std::memory_order_acquire);
        if (h == t) return;  // stopping
      }
    }
    for (; h < t; ++h) {
      LaunchJob& j = ring[h % kRing];
      lp.stream = stream;
      lp.grid = j.grid;
      lp.block = j.block;
      lp.rank = j.rank;
      lp.nargs = j.nargs;
      lp.shared_bytes = j.shared_bytes;
      lp.offset = j.offset;
      lp.global = j.global;
      for (unsigned i = 0; i < j.nargs; ++i) {
        const LaunchArg& a = i < kInlineArgs ? j.args[i] : j.more[i - kInlineArgs];
        lp.ptr[i] = a.ptr;
        lp.len[i] = a.len;
        lp.smem_offset[i] = a.smem_offset;
        lp.scalar[i] = a.scalar;
      }
      const int rc = j.launch(lp);
      if (rc != 0) finish_event(j.ev, false, "kernel " + j.name_copy + ": " + ndx_error_string(rc));
      // drop what the job holds now (a launcher may own device resources
      // that must not outlive the Device)
      j.ev.reset();
      j.launch = nullptr;
      j.more.reset();
      launched.store(j.seq, std::memory_order_release);
      q_done.store(h + 1, std::memory_order_release);
    }
  }
}

void DeviceImpl::watch(const std::shared_ptr<Event::State>& st) {
  const std::uint64_t s = st->seq.load(std::memory_order_acquire);
  if (s != 0 && completed.load(std::memory_order_acquire) >= s) {
    finish_event(st, true, {});
    return;
  }
  {
    std::lock_guard<std::mutex> l(watch_mu);
    watched.emplace(s, st);
  }
  watch_cv.notify_one();
}

void DeviceImpl::complete_upto(std::uint64_t s) {
  std::uint64_t prev = completed.load();
  while (prev < s && !completed.compare_exchange_weak(prev, s)) {
  }
  std::vector<std::shared_ptr<Event::State>> done;
  {
    std::lock_guard<std::mutex> l(watch_mu);
    auto end = watched.upper_bound(s);
    for (auto it = watched.begin(); it != end; ++it) done.push_back(it->second);
    watched.erase(watched.begin(), end);
  }
  for (auto& st : done) finish_event(st, true, {});
}

void DeviceImpl::fail_all(const std::string& why) {
  std::vector<std::shared_ptr<Event::State>> all;
  {
    std::lock_guard<std::mutex> l(watch_mu);
    for (auto& kv : watched) all.push_back(kv.second);
    watched.clear();
  }
  for (auto& st : all) finish_event(st, false, why);
}

bool DeviceImpl::sync_now() {
  std::uint64_t s;
  void* ev = nullptr;
  int rc = 0;
  {
    std::lock_guard<std::mutex> l(issue_mu);
    if (broken) {
      rc = -1;
    } else {
      drain();
      s = issued;
      rc = bind_thread(ordinal);
      if (!rc) rc = ndx_event_create(&ev, 0);
      if (!rc) rc = ndx_event_record(ev, stream);
    }
  }
  if (rc == 0) rc = ndx_event_synchronize(ev);
  if (ev) ndx_event_destroy(ev);
  if (rc != 0) {
    std::string why;
    {
      std::lock_guard<std::mutex> l(issue_mu);
      if (!broken) {
        broken = true;
        broken_why = "device failure: " + cuda_msg(rc);
      }
      why = broken_why;
    }
    fail_all(why);
    return false;
  }
  complete_upto(s);
  return true;
}

void DeviceImpl::poll() {
  std::uint64_t s;
  int rc;
  {
    std::lock_guard<std::mutex> l(issue_mu);
    if (broken) return;
    s = launched.load(std::memory_order_acquire);  // queued launches are not on the stream yet
    rc = bind_thread(ordinal);
    if (!rc) rc = ndx_stream_query(stream);
  }
  if (rc == 0) {
    complete_upto(s);
  } else if (rc != 1) {
    {
      std::lock_guard<std::mutex> l(issue_mu);
      broken = true;
      broken_why = "device failure: " + cuda_msg(rc);
    }
    fail_all("device failure: " + cuda_msg(rc));
  }
}

void DeviceImpl::completer_loop() {
  for (;;) {
    {
      std::unique_lock<std::mutex> l(watch_mu);
      watch_cv.wait(l, [&] { return stopping || !watched.empty(); });
      if (stopping && watched.empty()) return;
      if (stopping) {
        l.unlock();
        sync_now();
        continue;
      }
    }
    sync_now();
  }
}

void* DeviceImpl::pinned_get(std::size_t bytes, std::size_t& cap) {
  cap = 4096;
  while (cap < bytes) cap <<= 1;
  {
    std::lock_guard<std::mutex> l(pin_mu);
    auto it = pinned_free.find(cap);
    if (it != pinned_free.end()) {
      void* p = it->second;
      pinned_free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (ndx_host_alloc(&p, cap) != 0) return nullptr;
  return p;
}

std::size_t DeviceImpl::size_class(std::size_t bytes) {
  // 1/8-octave classes: at most 12.5% slack, few distinct classes
  if (bytes <= 4096) return 4096;
  std::size_t p = std::size_t(1) << (63 - __builtin_clzll(bytes - 1));  // <= bytes-1
  const std::size_t step = p / 8;
  return (bytes + step - 1) / step * step;
}

void* DeviceImpl::block_get(std::size_t cls) {
  auto it = block_cache.find(cls);
  if (it == block_cache.end()) return nullptr;
  void* p = it->second;
  block_cache.erase(it);
  cached_bytes -= cls;
  return p;
}

void DeviceImpl::block_put(void* p, std::size_t cls) {
  block_cache.emplace(cls, p);
  cached_bytes += cls;
  while (cached_bytes > kCacheLimit && !block_cache.empty()) {
    drain();
    bind_thread(ordinal);
    auto it = std::prev(block_cache.end());  // drop the largest
    ndx_free_async(it->second, stream);
    cached_bytes -= it->first;
    block_cache.erase(it);
  }
}

void DeviceImpl::block_trim() {
  drain();
  bind_thread(ordinal);
  for (auto& kv : block_cache) ndx_free_async(kv.second, stream);
  block_cache.clear();
  cached_bytes = 0;
}

void DeviceImpl::pinned_put(void* p, std::size_t cap) {
  std::lock_guard<std::mutex> l(pin_mu);
  pinned_free.emplace(cap, p);
}

}  // namespace detail

using detail::bind_thread;
using detail::DeviceImpl;

namespace {

struct Issue {
  std::string name;
  std::function<int(void*)> fn;     // issues the work on the stream
  std::vector<Event> other_device;  // pending deps issued on other devices
};

void check_deps(const std::vector<Event>& deps) {
  for (const Event& e : deps)
    if (!e.valid()) throw DeviceError("invalid dependency event");
}

// Issue `w` on the stream now; binds the event to the new stream position.
void issue_now(const std::shared_ptr<DeviceImpl>& d, const Event& ev, Issue& w) {
  std::lock_guard<std::mutex> l(d->issue_mu);
  if (d->broken) {
    detail::finish_event(ev.shared_state(), false, d->broken_why);
    return;
  }
  d->drain();
  for (const Event& dep : w.other_device) {
    auto od = dep.shared_state()->dev.lock();
    if (!od) continue;
    // the dependency may still sit in the other device's launch ring: the
    // fence must follow its actual launch
    const std::uint64_t want = dep.shared_state()->seq.load(std::memory_order_acquire);
    for (unsigned i = 0; od->launched.load(std::memory_order_acquire) < want; ++i)
      if (i > 256) std::this_thread::yield();
    // the fence event belongs to the producer's device and is recorded on
    // its stream; the consumer's stream then waits on it (cross-device wait)
    void* fence = nullptr;
    int frc = bind_thread(od->ordinal);
    if (!frc) frc = ndx_event_create(&fence, 0);
    if (!frc) frc = ndx_event_record(fence, od->stream);
    const int brc = bind_thread(d->ordinal);
    if (!frc) frc = brc;
    if (!frc) frc = ndx_stream_wait_event(d->stream, fence);
    if (fence) ndx_event_destroy(fence);
    if (frc) {
      detail::finish_event(ev.shared_state(), false,
                           "kernel " + w.name + ": cross-device fence: " + ndx_error_string(frc));
      return;
    }
  }
  if (const int brc = bind_thread(d->ordinal)) {
    detail::finish_event(ev.shared_state(), false, "kernel " + w.name + ": " + ndx_error_string(brc));
    return;
  }
  ev.mark_exec_start();
  const int rc = w.fn(d->stream);
  if (rc != 0) {
    detail::finish_event(ev.shared_state(), false, "kernel " + w.name + ": " + ndx_error_string(rc));
    return;
  }
  auto& es = *ev.shared_state();
  es.seq.store(++d->issued, std::memory_order_release);
  d->launched.store(d->issued, std::memory_order_release);
  bool waited;
  {
    std::lock_guard<std::mutex> lk(es.mu);
    waited = !es.callbacks.empty() || es.awaited;
  }
  if (waited) d->watch(ev.shared_state());  // callbacks registered while deferred
}

// The reference admits commands in order and runs them once their
// dependencies are terminal (device.cpp:61-105).  Same-device dependencies
// are satisfied by stream order; the rest defer the issue.
Event submit(const std::shared_ptr<DeviceImpl>& d, Issue w, const std::vector<Event>& deps) {
  Event ev = detail::make_device_event(d);
  std::vector<Event> wait;
  for (const Event& dep : deps) {
    EventState st;
    {
      // peek without polling the stream: the hot path must stay API-free
      std::lock_guard<std::mutex> l(dep.shared_state()->mu);
      st = dep.shared_state()->st;
    }
    if (st == EventState::failed) {
      detail::finish_event(ev.shared_state(), false, "dependency failed");
      return ev;
    }
    if (st == EventState::complete) continue;
    auto ds = dep.shared_state();
    auto dd = ds->dev.lock();
    if (dd && ds->seq.load(std::memory_order_acquire) != 0) {
      if (dd != d) w.other_device.push_back(dep);
      continue;  // issued earlier on a stream: ordering by stream / fence
    }
    wait.push_back(dep);  // host event or not yet issued
  }
  if (wait.empty()) {
    issue_now(d, ev, w);
    return ev;
  }
  {
    std::lock_guard<std::mutex> l(d->defer_mu);
    ++d->deferred;
  }
  struct Pending {
    std::atomic<int> left;
    std::atomic<bool> failed{false};
    Issue w;
  };
  auto pend = std::make_shared<Pending>();
  pend->left.store(int(wait.size()));
  pend->w = std::move(w);
  for (const Event& dep : wait) {
    dep.add_callback([d, ev, pend](EventState s) {
      if (s == EventState::failed) pend->failed.store(true);
      if (pend->left.fetch_sub(1) != 1) return;
      if (pend->failed.load())
        detail::finish_event(ev.shared_state(), false, "dependency failed");
      else
        issue_now(d, ev, pend->w);
      {
        std::lock_guard<std::mutex> l(d->defer_mu);
        --d->deferred;
      }
      d->defer_cv.notify_all();
    });
  }
  return ev;
}

void check_target(const Device* self, const Buffer& b) {
  if (!b.valid()) throw DeviceError("invalid buffer");
  if (&b.device() != self) throw DeviceError("buffer belongs to a different device");
  if (b.freed()) throw DeviceError("buffer already freed");
}

}  // namespace

Device::Device(DeviceConfig cfg) : cfg_(cfg), impl_(std::make_shared<DeviceImpl>()) {
  if (cfg_.max_group_size == 0) throw DeviceError("group size cap must be positive");
  if (cfg_.max_group_size > 1024) cfg_.max_group_size = 1024;
  int rc = ndx_device_open(cfg_.ordinal);
  if (rc != 0) throw DeviceError(std::string("cannot open CUDA device: ") + ndx_error_string(rc));
  impl_->ordinal = cfg_.ordinal;
  impl_->max_group = cfg_.max_group_size;
  rc = ndx_stream_create(&impl_->stream);
  if (rc != 0) throw DeviceError(std::string("cannot create stream: ") + ndx_error_string(rc));
  impl_->start();
}

Device::~Device() {
  try {
    await_all();
  } catch (...) {
  }
  impl_->stop();
  {
    std::lock_guard<std::mutex> l(impl_->issue_mu);
    impl_->block_trim();
  }
  {
    std::lock_guard<std::mutex> l(impl_->pin_mu);
    for (auto& kv : impl_->pinned_free) ndx_host_free(kv.second);
    impl_->pinned_free.clear();
  }
  ndx_stream_synchronize(impl_->stream);
  ndx_stream_destroy(impl_->stream);
}

void* Device::stream() const {
  std::lock_guard<std::mutex> l(impl_->issue_mu);
  impl_->drain();  // everything enqueued so far is on the stream
  return impl_->stream;
}

namespace {
Buffer make_buffer(Device* self, const std::shared_ptr<DeviceImpl>& d, ElemType type,
                   std::int64_t length, Access access, bool zero) {
  if (length < 0) throw DeviceError("buffer length is negative");
  auto st = std::make_shared<detail::BufferState>();
  st->id = d->next_buffer_id.fetch_add(1);
  st->type = type;
  st->length = std::size_t(length);
  st->access = access;
  st->device = self;
  const std::size_t bytes = std::max<std::size_t>(st->length * elem_size(type), 16);
  const std::size_t cls = DeviceImpl::size_class(bytes);
  {
    std::lock_guard<std::mutex> l(d->issue_mu);
    int rc = 0;
    st->ptr = d->block_get(cls);
    if (!st->ptr || zero) d->drain();
    if (!st->ptr) {
      rc = ndx_malloc_async(&st->ptr, cls, d->stream);
      if (rc != 0) {  // out of memory: give the cache back and retry once
        d->block_trim();
        rc = ndx_malloc_async(&st->ptr, cls, d->stream);
      }
    }
    if (rc == 0 && zero) rc = ndx_memset_async(st->ptr, 0, bytes, d->stream);
    if (rc != 0) throw DeviceError(std::string("device allocation failed: ") + ndx_error_string(rc));
  }
  d->live.fetch_add(1);
  return Buffer(std::move(st));
}
}  // namespace

Buffer Device::create_buffer(ElemType type, std::int64_t length, Access access) {
  return make_buffer(this, impl_, type, length, access, true);
}

Buffer Device::create_buffer_uninit(ElemType type, std::int64_t length, Access access) {
  return make_buffer(this, impl_, type, length, access, false);
}

Buffer Device::wrap_buffer(void* device_ptr, ElemType type, std::int64_t length, Access access) {
  if (length < 0) throw DeviceError("buffer length is negative");
  if (!device_ptr && length > 0) throw DeviceError("null device pointer");
  auto st = std::make_shared<detail::BufferState>();
  st->id = impl_->next_buffer_id.fetch_add(1);
  st->type = type;
  st->length = std::size_t(length);
  st->access = access;
  st->device = this;
  st->ptr = device_ptr;
  st->owned = false;
  impl_->live.fetch_add(1);
  return Buffer(std::move(st));
}

void Device::free_buffer(const Buffer& b) {
  if (!b.valid()) throw DeviceError("invalid buffer");
  if (&b.device() != this) throw DeviceError("buffer belongs to a different device");
  if (b.state().freed.exchange(true, std::memory_order_acq_rel))
    throw DeviceError("buffer already freed");
  impl_->live.fetch_sub(1);
  // Release in stream order: commands already issued still see the storage.
  // A command deferred on a host event holds the BufferState and keeps
  // `ptr` valid because the stream-ordered free lands after it is issued
  // only if it was issued first -- deferred commands therefore re-check
  // `freed` and fail instead of touching released memory.
  if (!b.state().owned) return;
  std::lock_guard<std::mutex> l(impl_->issue_mu);
  const std::size_t bytes = std::max<std::size_t>(b.bytes(), 16);
  impl_->block_put(b.state().ptr, DeviceImpl::size_class(bytes));
}

std::size_t Device::live_buffers() const { return impl_->live.load(); }

Event Device::enqueue_write_bytes(const Buffer& b, std::vector<std::byte> data,
                                  std::vector<Event> deps) {
  check_target(this, b);
  check_deps(deps);
  if (data.size() != b.bytes()) throw DeviceError("write size does not match the buffer");
  auto st = b.shared_state();
  auto bytes = std::make_shared<std::vector<std::byte>>(std::move(data));
  Issue w{"write", [st, bytes](void* s) -> int {
            if (st->freed.load()) return NDX_E_INVALID;
            return ndx_memcpy_h2d_async(st->ptr, bytes->data(), bytes->size(), s);
          }, {}};
  return submit(impl_, std::move(w), deps);
}

Event Device::enqueue_write_from(const Buffer& b, const void* src, std::size_t bytes,
                                 std::vector<Event> deps) {
  check_target(this, b);
  check_deps(deps);
  if (bytes != b.bytes()) throw DeviceError("write size does not match the buffer");
  if (!src && bytes) throw DeviceError("write source is null");
  auto st = b.shared_state();
  Issue w{"write", [st, src, bytes](void* s) -> int {
            if (st->freed.load()) return NDX_E_INVALID;
            return bytes ? ndx_memcpy_h2d_async(st->ptr, src, bytes, s) : 0;
          }, {}};
  return submit(impl_, std::move(w), deps);
}

Event Device::enqueue_read_into(const Buffer& b, void* dst, std::size_t nbytes, std::vector<Event> deps) {
  if (!dst && nbytes) throw DeviceError("read destination is null");
  return enqueue_read_with(
      b, nbytes, [dst](const void* p, std::size_t k) { if (k) std::memcpy(dst, p, k); }, std::move(deps));
}

Event Device::enqueue_read_with(const Buffer& b, std::size_t nbytes,
                                std::function<void(const void*, std::size_t)> consume,
                                std::vector<Event> deps) {
  check_target(this, b);
  check_deps(deps);
  if (nbytes > b.bytes()) throw DeviceError("read size exceeds the buffer");
  auto st = b.shared_state();
  auto d = impl_;
  struct Stage {
    void* pinned = nullptr;
    std::size_t cap = 0;
  };
  auto stage = std::make_shared<Stage>();
  stage->pinned = d->pinned_get(std::max<std::size_t>(nbytes, 1), stage->cap);
  if (!stage->pinned) throw DeviceError("cannot allocate pinned staging memory");
  Issue w{"read", [st, stage, nbytes](void* s) -> int {
            if (st->freed.load()) return NDX_E_INVALID;
            return nbytes ? ndx_memcpy_d2h_async(stage->pinned, st->ptr, nbytes, s) : 0;
          }, {}};
  Event ev = detail::make_device_event(d);
  ev.shared_state()->before_complete = [d, stage, nbytes, consume = std::move(consume)] {
    consume(stage->pinned, nbytes);
    d->pinned_put(stage->pinned, stage->cap);
  };
  Event issued = submit(d, std::move(w), deps);
  auto es = ev.shared_state();
  issued.add_callback([es, issued](EventState s) {
    detail::finish_event(es, s == EventState::complete, s == EventState::complete ? "" : issued.error());
  });
  return ev;
}

Event Device::enqueue_read_bytes(const Buffer& b, std::shared_ptr<std::vector<std::byte>> dst,
                                 std::vector<Event> deps) {
  check_target(this, b);
  check_deps(deps);
  if (!dst) throw DeviceError("read destination is null");
  auto st = b.shared_state();
  auto d = impl_;
  const std::size_t nbytes = b.bytes();
  struct Stage {
    void* pinned = nullptr;
    std::size_t cap = 0;
  };
  auto stage = std::make_shared<Stage>();
  stage->pinned = d->pinned_get(std::max<std::size_t>(nbytes, 1), stage->cap);
  if (!stage->pinned) throw DeviceError("cannot allocate pinned staging memory");
  Issue w{"read", [st, stage, nbytes](void* s) -> int {
            if (st->freed.load()) return NDX_E_INVALID;
            return ndx_memcpy_d2h_async(stage->pinned, st->ptr, nbytes, s);
          }, {}};
  Event ev = detail::make_device_event(d);
  // the copy into the caller's vector happens before the event completes
  ev.shared_state()->before_complete = [d, stage, dst, nbytes] {
    dst->resize(nbytes);
    if (nbytes) std::memcpy(dst->data(), stage->pinned, nbytes);
    d->pinned_put(stage->pinned, stage->cap);
  };
  // route through submit with a pre-made event
  Event issued = submit(d, std::move(w), deps);
  // forward the terminal state of `issued` into `ev` (after the copy)
  auto es = ev.shared_state();
  issued.add_callback([es, issued](EventState s) {
    detail::finish_event(es, s == EventState::complete, s == EventState::complete ? "" : issued.error());
  });
  return ev;
}

Event Device::enqueue_kernel(const KernelDef& kernel, NdRange range, std::vector<KernelArg> args,
                             std::vector<Event> deps) {
  if (!kernel.launch) throw DeviceError("kernel has no launcher");
  if (args.size() > LaunchParams::kMaxArgs) throw DeviceError("too many kernel arguments");
  check_deps(deps);
  for (const KernelArg& a : args)
    if (a.kind == KernelArg::Kind::global) check_target(this, a.buffer);
  const auto local = resolve_local(range, cfg_.max_group_size);

  LaunchParams p;
  p.rank = range.rank;
  p.offset = range.offset;
  p.global = range.global;
  for (int d = 0; d < 3; ++d) {
    p.block[d] = unsigned(local[d]);
    p.grid[d] = unsigned(range.global[d] / local[d]);
  }
  p.nargs = args.size();
  std::size_t smem = 0;
  for (std::size_t i = 0; i < args.size(); ++i) {
    const KernelArg& a = args[i];
    switch (a.kind) {
      case KernelArg::Kind::global:
        p.ptr[i] = a.buffer.data();
        p.len[i] = a.buffer.length();
        break;
      case KernelArg::Kind::local:
        smem = (smem + 15) & ~std::size_t(15);
        p.smem_offset[i] = smem;
        p.len[i] = a.local_len;
        smem += a.local_len * elem_size(a.local_type);
        break;
      case KernelArg::Kind::scalar:
        p.scalar[i] = a.value;
        break;
    }
  }
  p.shared_bytes = smem;

  // Fast path: every dependency is complete or issued earlier on this
  // device's stream -> launch right here, nothing allocated for the command.
  bool direct = true;
  for (const Event& dep : deps) {
    auto& ds = *dep.shared_state();
    EventState st;
    {
      std::lock_guard<std::mutex> l(ds.mu);
      st = ds.st;
    }
    if (st == EventState::complete) continue;
    if (st == EventState::failed) {
      direct = false;
      break;
    }
    auto dd = ds.dev.lock();
    if (!(dd == impl_ && ds.seq.load(std::memory_order_acquire) != 0)) {
      direct = false;
      break;
    }
  }
  if (direct) {
    Event ev = detail::make_device_event(impl_);
    std::lock_guard<std::mutex> l(impl_->issue_mu);
    if (impl_->broken) {
      detail::finish_event(ev.shared_state(), false, impl_->broken_why);
      return ev;
    }
    // stream position now, the launch itself on the launcher thread
    const std::uint64_t seq = ++impl_->issued;
    ev.mark_exec_start();  // handed to the stream's launcher now
    ev.shared_state()->seq.store(seq, std::memory_order_release);
    impl_->push_launch(p, kernel.launch, ev.shared_state(), seq, kernel.name);
    return ev;
  }

  std::vector<std::shared_ptr<detail::BufferState>> bufs;
  for (const KernelArg& a : args)
    if (a.kind == KernelArg::Kind::global) bufs.push_back(a.buffer.shared_state());
  auto pp = std::make_shared<LaunchParams>(p);
  Launcher launch = kernel.launch;
  Issue w{kernel.name, [pp, launch, bufs](void* s) -> int {
            for (auto& b : bufs)
              if (b->freed.load()) return NDX_E_INVALID;  // freed while deferred
            pp->stream = s;
            return launch(*pp);
          }, {}};
  return submit(impl_, std::move(w), deps);
}

Event Device::enqueue_native(std::string name, std::function<int(void*)> fn,
                             std::vector<Event> deps) {
  check_deps(deps);
  Issue w{std::move(name), std::move(fn), {}};
  return submit(impl_, std::move(w), deps);
}

void Device::await_all() {
  {
    std::unique_lock<std::mutex> l(impl_->defer_mu);
    impl_->defer_cv.wait(l, [&] { return impl_->deferred == 0; });
  }
  impl_->sync_now();
}

}  // namespace ndactor
