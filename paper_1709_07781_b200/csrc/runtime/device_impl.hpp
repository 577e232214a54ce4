// Internal: the CUDA device behind ndactor::Device and the Event state.
#pragma once

#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ndactor/device.hpp"
#include "ndactor/event.hpp"
#include "ndactor/kernel.hpp"

namespace ndactor {

struct Event::State {
  std::uint64_t id = 0;
  std::mutex mu;
  std::condition_variable cv;
  EventState st = EventState::pending;
  std::string error;
  std::vector<Callback> callbacks;
  Clock::time_point enqueue_tp = Clock::now();
  Clock::time_point exec_start_tp{};
  Clock::time_point terminal_tp{};
  std::atomic<bool> exec_started{false};
  // device binding: the stream position (0 = not issued on a device yet)
  std::weak_ptr<detail::DeviceImpl> dev;
  std::atomic<std::uint64_t> seq{0};
  bool awaited = false;  // someone blocks in await() (guarded by mu)
  // runs on the completing thread right before the terminal transition
  std::function<void()> before_complete;
};

namespace detail {

// Make `ordinal` the calling host thread's current CUDA device (cached per
// thread); 0 or a CUDA error code.
int bind_thread(int ordinal);

struct DeviceImpl : std::enable_shared_from_this<DeviceImpl> {
  int ordinal = 0;
  void* stream = nullptr;
  std::size_t max_group = 1024;

  // issue order == stream order == sequence order
  std::mutex issue_mu;
  std::uint64_t issued = 0;
  bool broken = false;
  std::string broken_why;

  // completion tracking
  std::mutex watch_mu;
  std::condition_variable watch_cv;
  std::multimap<std::uint64_t, std::shared_ptr<Event::State>> watched;
  std::atomic<std::uint64_t> completed{0};
  bool stopping = false;
  std::thread completer;

  // commands waiting on host events / unissued dependencies
  std::mutex defer_mu;
  std::condition_variable defer_cv;
  std::size_t deferred = 0;

  // Launch pipeline.  Kernels on the direct path (every dependency already
  // on this stream) get their stream position at enqueue time and are handed,
  // in that order, to one launcher thread: the enqueuing thread (an actor)
  // goes on with its message while the ~2.5 us cudaLaunchKernel runs on
  // another core.  Every other stream operation first drains the queue, so
  // issue order stays stream order.
  // A queued launch, packed so that the few cache lines it spans are all the
  // launcher core has to pull from the enqueuing core (the LaunchParams the
  // kernel's launcher sees is rebuilt in the launcher thread's own copy).
  struct LaunchArg {
    void* ptr;
    std::size_t len;
    std::size_t smem_offset;
    Scalar scalar;
  };
  static constexpr std::size_t kInlineArgs = 2;
  struct alignas(64) LaunchJob {
    std::uint64_t seq = 0;
    std::shared_ptr<Event::State> ev;
    Launcher launch;
    std::array<unsigned, 3> grid{}, block{};
    unsigned rank = 1;
    unsigned nargs = 0;
    std::size_t shared_bytes = 0;
    std::array<std::size_t, 3> offset{}, global{};
    LaunchArg args[kInlineArgs];
    std::unique_ptr<LaunchArg[]> more;  // arguments past kInlineArgs
    std::string name_copy;
  };
  // single-producer (under issue_mu) / single-consumer ring: a push copies
  // only the arguments the kernel has, so little crosses between cores
  static constexpr std::size_t kRing = 8192;
  std::unique_ptr<LaunchJob[]> ring{new LaunchJob[kRing]};
  std::mutex q_mu;
  std::condition_variable q_cv;
  bool q_stop = false;
  std::atomic<bool> q_sleeping{false};
  std::atomic<std::uint64_t> q_pushed{0}, q_done{0};
  std::atomic<std::uint64_t> launched{0};  // stream position actually issued
  std::thread launcher;
  void launcher_loop();
  // caller holds issue_mu
  void push_launch(const LaunchParams& p, const Launcher& launch,
                   const std::shared_ptr<Event::State>& ev, std::uint64_t seq, const std::string& name);
  void drain();                     // caller holds issue_mu: every pushed job issued

  std::atomic<std::size_t> live{0};
  std::atomic<std::uint64_t> next_buffer_id{1};

  // pinned staging blocks for asynchronous reads, by power-of-two size
  std::mutex pin_mu;
  std::multimap<std::size_t, void*> pinned_free;

  // Device blocks released by free_buffer, kept for reuse by size class.
  // Frees and allocations are both ordered on the one stream, so handing a
  // released block to the next allocation is safe without any wait -- the
  // same rule stream-ordered pools follow, minus their per-call cost for
  // multi-GB blocks.  Guarded by issue_mu.
  std::multimap<std::size_t, void*> block_cache;
  std::size_t cached_bytes = 0;
  static constexpr std::size_t kCacheLimit = std::size_t(64) << 30;
  static std::size_t size_class(std::size_t bytes);
  void* block_get(std::size_t cls);
  void block_put(void* p, std::size_t cls);
  void block_trim();

  void start();
  void stop();
  /// Completes every watched event with seq <= s (runs callbacks).
  void complete_upto(std::uint64_t s);
  void fail_all(const std::string& why);
  /// Blocks until everything issued so far is done; returns false on a
  /// sticky device error (then every pending event has been failed).
  bool sync_now();
  /// Non-blocking progress check used by Event::state().
  void poll();
  void watch(const std::shared_ptr<Event::State>& st);
  void completer_loop();

  void* pinned_get(std::size_t bytes, std::size_t& cap);
  void pinned_put(void* p, std::size_t cap);
};

Event make_device_event(const std::shared_ptr<DeviceImpl>& d);
void finish_event(const std::shared_ptr<Event::State>& st, bool ok, std::string why);

}  // namespace detail
}  // namespace ndactor
