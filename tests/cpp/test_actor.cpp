// Actor runtime contract, restating p/tests/test_actor.cpp:24-320 (CPU only).
#include <atomic>
#include <map>
#include <thread>

#include "harness.hpp"
#include "ndactor/actor.hpp"

using namespace ndactor;

namespace {
ActorHandle summer(ActorSystem& sys) {
  Behavior b;
  b.on({ValueKind::i64, ValueKind::i64}, [](Context&, Message m) {
    return HandlerResult::reply(Message::of(m.at(0).as_i64() + m.at(1).as_i64()));
  });
  return sys.spawn(std::move(b));
}
std::int64_t i64_of(const Reply& r) { return get_message(r).at(0).as_i64(); }
}  // namespace

TEST("cpu", "actor: request gets the handler's reply") {
  ActorSystem sys(3);
  auto a = summer(sys);
  Reply r = sys.request(a, Message::of(std::int64_t{19}, std::int64_t{23})).await();
  REQUIRE(!is_error(r));
  CHECK(i64_of(r) == 42);
}

TEST("cpu", "actor: unmatched message is a mismatch error") {
  ActorSystem sys(2);
  Reply r = sys.request(summer(sys), Message::of(1.5)).await();
  REQUIRE(is_error(r));
  CHECK(get_error(r).code == ErrorCode::mismatch);
}

TEST("cpu", "actor: clauses are tried in registration order") {
  ActorSystem sys(2);
  Behavior b;
  b.on({ValueKind::i64}, [](Context&, Message) { return HandlerResult::reply(Message::of(std::int64_t{7})); });
  b.otherwise([](Context&, Message) { return HandlerResult::reply(Message::of(std::int64_t{8})); });
  auto a = sys.spawn(std::move(b));
  CHECK(i64_of(sys.request(a, Message::of(std::int64_t{0})).await()) == 7);
  CHECK(i64_of(sys.request(a, Message::of(2.0)).await()) == 8);
}

TEST("cpu", "actor: handler exceptions become unhandled errors, actor survives") {
  ActorSystem sys(2);
  Behavior b;
  b.on({ValueKind::i64}, [](Context&, Message) -> HandlerResult { throw std::runtime_error("bang"); });
  auto a = sys.spawn(std::move(b));
  Reply r = sys.request(a, Message::of(std::int64_t{1})).await();
  REQUIRE(is_error(r));
  CHECK(get_error(r).code == ErrorCode::unhandled);
  CHECK(get_error(r).what == "bang");
  CHECK(is_error(sys.request(a, Message::of(std::int64_t{1})).await()));
}

TEST("cpu", "actor: one worker at a time, per-sender FIFO") {
  ActorSystem sys(8);
  std::atomic<bool> inside{false};
  std::atomic<int> overlaps{0}, breaks{0}, handled{0};
  auto last = std::make_shared<std::map<std::int64_t, std::int64_t>>();
  Behavior b;
  b.on({ValueKind::i64, ValueKind::i64}, [&, last](Context&, Message m) {
    if (inside.exchange(true)) overlaps.fetch_add(1);
    const std::int64_t s = m.at(0).as_i64(), q = m.at(1).as_i64();
    auto it = last->find(s);
    if ((it == last->end() ? -1 : it->second) != q - 1) breaks.fetch_add(1);
    (*last)[s] = q;
    handled.fetch_add(1);
    inside.store(false);
    return HandlerResult::no_reply();
  });
  auto probe = sys.spawn(std::move(b));
  std::vector<std::thread> ts;
  for (int s = 0; s < 6; ++s)
    ts.emplace_back([&, s] {
      for (std::int64_t q = 0; q < 400; ++q) sys.send(probe, Message::of(std::int64_t{s}, q));
    });
  for (auto& t : ts) t.join();
  sys.await_idle();
  CHECK(overlaps.load() == 0);
  CHECK(breaks.load() == 0);
  CHECK(handled.load() == 6 * 400);
}

TEST("cpu", "actor: become swaps the behavior") {
  ActorSystem sys(2);
  Behavior second;
  second.on({ValueKind::i64}, [](Context&, Message) { return HandlerResult::reply(Message::of(std::int64_t{2})); });
  Behavior first;
  first.on({ValueKind::i64}, [second](Context&, Message) {
    return HandlerResult::reply(Message::of(std::int64_t{1})).and_become(second);
  });
  auto a = sys.spawn(std::move(first));
  CHECK(i64_of(sys.request(a, Message::of(std::int64_t{0})).await()) == 1);
  CHECK(i64_of(sys.request(a, Message::of(std::int64_t{0})).await()) == 2);
}

TEST("cpu", "actor: delegation hands the reply obligation on") {
  ActorSystem sys(2);
  auto target = summer(sys);
  Behavior b;
  b.otherwise([target](Context&, Message m) { return HandlerResult::delegate(target, std::move(m)); });
  auto front = sys.spawn(std::move(b));
  CHECK(i64_of(sys.request(front, Message::of(std::int64_t{5}, std::int64_t{6})).await()) == 11);
}

TEST("cpu", "actor: taken promise answers later; dropped promise breaks") {
  ActorSystem sys(2);
  std::shared_ptr<ReplyPromise> kept = std::make_shared<ReplyPromise>();
  Behavior b;
  b.on({ValueKind::i64}, [kept](Context& ctx, Message) {
    *kept = ctx.take_promise();
    return HandlerResult::reply(Message::of(std::int64_t{-1}));  // ignored: promise taken
  });
  b.on({ValueKind::f64}, [](Context& ctx, Message) {
    ctx.take_promise();  // dropped on the floor
    return HandlerResult::no_reply();
  });
  auto a = sys.spawn(std::move(b));
  ResponseHandle h = sys.request(a, Message::of(std::int64_t{1}));
  sys.await_idle();
  kept->deliver(Message::of(std::int64_t{99}));
  CHECK(i64_of(h.await()) == 99);
  Reply broken = sys.request(a, Message::of(1.0)).await();
  REQUIRE(is_error(broken));
  CHECK(get_error(broken).code == ErrorCode::broken_promise);
}

TEST("cpu", "actor: exit, down errors, monitors fire once, terminate") {
  ActorSystem sys(2);
  Behavior b;
  b.on({ValueKind::i64}, [](Context&, Message) { return HandlerResult::no_reply().and_exit(); });
  auto a = sys.spawn(std::move(b));
  std::atomic<int> downs{0};
  Behavior ob;
  ob.on_opaque<DownMsg>(std::function<HandlerResult(Context&, DownMsg)>([&](Context&, DownMsg) {
    downs.fetch_add(1);
    return HandlerResult::no_reply();
  }));
  auto obs = sys.spawn(std::move(ob));
  sys.monitor(a, obs);
  sys.send(a, Message::of(std::int64_t{1}));
  sys.await_idle();
  Reply r = sys.request(a, Message::of(std::int64_t{1})).await();
  REQUIRE(is_error(r));
  CHECK(get_error(r).code == ErrorCode::down);
  sys.monitor(a, obs);  // already down: delivered immediately
  sys.await_idle();
  CHECK(downs.load() == 2);

  auto t = summer(sys);
  sys.terminate(t);
  sys.await_idle();
  Reply rt = sys.request(t, Message::of(std::int64_t{1}, std::int64_t{2})).await();
  CHECK(is_error(rt) && get_error(rt).code == ErrorCode::down);
  CHECK(sys.live_actors() >= 1);
}

TEST("cpu", "actor: compose pipes inner reply into outer, errors pass through") {
  ActorSystem sys(4);
  Behavior dbl;
  dbl.on({ValueKind::i64}, [](Context&, Message m) {
    if (m.at(0).as_i64() < 0) return HandlerResult::error(ErrorCode::unhandled, "negative");
    return HandlerResult::reply(Message::of(2 * m.at(0).as_i64()));
  });
  Behavior inc;
  inc.on({ValueKind::i64}, [](Context&, Message m) { return HandlerResult::reply(Message::of(m.at(0).as_i64() + 1)); });
  auto f = sys.spawn(std::move(dbl)), g = sys.spawn(std::move(inc));
  auto gf = g * f;  // f first
  auto fg = f * g;
  CHECK(i64_of(sys.request(gf, Message::of(std::int64_t{5})).await()) == 11);
  CHECK(i64_of(sys.request(fg, Message::of(std::int64_t{5})).await()) == 12);
  Reply e = sys.request(gf, Message::of(std::int64_t{-3})).await();
  REQUIRE(is_error(e));
  CHECK(get_error(e).what == "negative");
}

TEST("cpu", "actor: then() fires exactly once") {
  ActorSystem sys(2);
  std::atomic<int> fired{0};
  ResponseHandle h = sys.request(summer(sys), Message::of(std::int64_t{1}, std::int64_t{1}));
  h.then([&](Reply) { fired.fetch_add(1); });
  sys.await_idle();
  h.then([&](Reply) { fired.fetch_add(1); });  // already consumed
  CHECK(fired.load() == 1);
}
