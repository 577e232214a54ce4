// Event: completion token of a device command (reference: p/core/src/event.cpp).
#include "ndactor/event.hpp"

#include <atomic>
#include <utility>

#include "device_impl.hpp"

namespace ndactor {

namespace {
std::atomic<std::uint64_t> g_next_event{1};
}

Event Event::create() {
  auto s = std::make_shared<State>();
  s->id = g_next_event.fetch_add(1, std::memory_order_relaxed);
  return Event(std::move(s));
}

std::uint64_t Event::id() const { return state_->id; }

EventState Event::state() const {
  {
    std::lock_guard<std::mutex> l(state_->mu);
    if (state_->st != EventState::pending) return state_->st;
  }
  // a device command completes on the GPU without anybody being told:
  // look at the stream lazily
  if (state_->seq.load(std::memory_order_acquire) != 0) {
    if (auto d = state_->dev.lock()) {
      d->poll();
      if (d->completed.load(std::memory_order_acquire) >= state_->seq.load()) {
        detail::finish_event(state_, true, {});
      } else {
        bool broken;
        std::string why;
        {
          std::lock_guard<std::mutex> l(d->issue_mu);
          broken = d->broken;
          why = d->broken_why;
        }
        if (broken) detail::finish_event(state_, false, why);
      }
    }
  }
  std::lock_guard<std::mutex> l(state_->mu);
  return state_->st;
}

std::string Event::error() const {
  std::lock_guard<std::mutex> l(state_->mu);
  return state_->error;
}

void Event::add_callback(Callback fn) const {
  EventState st;
  {
    std::lock_guard<std::mutex> l(state_->mu);
    if (state_->st == EventState::pending) {
      state_->callbacks.push_back(std::move(fn));
      st = EventState::pending;
    } else {
      st = state_->st;
    }
  }
  if (st != EventState::pending) {
    fn(st);
    return;
  }
  // make sure somebody will complete it
  if (auto d = state_->dev.lock())
    if (state_->seq.load(std::memory_order_acquire) != 0) d->watch(state_);
}

EventState Event::await() const {
  {
    std::lock_guard<std::mutex> l(state_->mu);
    if (state_->st != EventState::pending) return state_->st;
    state_->awaited = true;  // a deferred command gets watched once issued
  }
  if (state_->seq.load(std::memory_order_acquire) != 0) {
    if (auto d = state_->dev.lock()) {
      d->watch(state_);
      d->sync_now();
    }
  }
  std::unique_lock<std::mutex> l(state_->mu);
  state_->cv.wait(l, [&] { return state_->st != EventState::pending; });
  return state_->st;
}

Clock::time_point Event::enqueue_time() const { return state_->enqueue_tp; }

Clock::time_point Event::exec_start_time() const {
  std::lock_guard<std::mutex> l(state_->mu);
  return state_->exec_start_tp;
}

Clock::time_point Event::terminal_time() const {
  std::lock_guard<std::mutex> l(state_->mu);
  return state_->terminal_tp;
}

void Event::mark_exec_start() const {
  if (state_->exec_started.exchange(true)) return;
  std::lock_guard<std::mutex> l(state_->mu);
  state_->exec_start_tp = Clock::now();
}

void Event::complete() const { detail::finish_event(state_, true, {}); }

void Event::fail(std::string reason) const { detail::finish_event(state_, false, std::move(reason)); }

namespace detail {

void finish_event(const std::shared_ptr<Event::State>& st, bool ok, std::string why) {
  std::function<void()> pre;
  {
    std::lock_guard<std::mutex> l(st->mu);
    if (st->st != EventState::pending) return;
    pre = std::move(st->before_complete);
    st->before_complete = nullptr;
  }
  if (pre && ok) pre();
  std::vector<Event::Callback> cbs;
  EventState fin = ok ? EventState::complete : EventState::failed;
  {
    std::lock_guard<std::mutex> l(st->mu);
    if (st->st != EventState::pending) return;
    if (!st->exec_started.exchange(true)) st->exec_start_tp = Clock::now();
    st->st = fin;
    if (!ok) st->error = std::move(why);
    st->terminal_tp = Clock::now();
    cbs.swap(st->callbacks);
  }
  st->cv.notify_all();
  for (auto& cb : cbs) cb(fin);
}

Event make_device_event(const std::shared_ptr<DeviceImpl>& d) {
  Event e = Event::create();
  e.shared_state()->dev = d;
  return e;
}

}  // namespace detail
}  // namespace ndactor
