// Device / MemRef / compute-actor / WAH device contract on a real GPU,
// restating p/tests/test_device.cpp, test_compute.cpp and test_wah_device.cpp.
// (NdRange resolution rules run in the "cpu" group.)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <numeric>
#include <random>
#include <thread>

#include "harness.hpp"
#include "ndactor/compute_actor.hpp"
#include "ndactor/mem_ref.hpp"
#include "ndactor/wah_device.hpp"
#include "ndactor/wah_io.hpp"

using namespace ndactor;

// ---- the oracle (test infrastructure only) --------------------------------
extern "C" {
typedef struct {
  uint32_t value, offset, length;
} wo_entry;
void* wo_reference_index(const uint32_t* values, uint64_t n);
uint32_t wo_index_row_count(const void*);
uint64_t wo_index_num_entries(const void*);
uint64_t wo_index_num_words(const void*);
const wo_entry* wo_index_entries(const void*);
const uint32_t* wo_index_words(const void*);
void wo_index_free(void*);
}

static wah::WahIndex oracle_index(const std::vector<uint32_t>& v) {
  void* h = wo_reference_index(v.data(), v.size());
  wah::WahIndex idx;
  idx.row_count = wo_index_row_count(h);
  const wo_entry* e = wo_index_entries(h);
  for (uint64_t i = 0; i < wo_index_num_entries(h); ++i) idx.entries.push_back({e[i].value, e[i].offset, e[i].length});
  const uint32_t* w = wo_index_words(h);
  idx.words.assign(w, w + wo_index_num_words(h));
  wo_index_free(h);
  return idx;
}

// ---- test kernels ----------------------------------------------------------
__global__ void k_square(const uint32_t* in, uint32_t* out, size_t n) {
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = in[i] * in[i];
}
__global__ void k_iota(uint32_t* out, size_t n) {
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = uint32_t(i);
}
__global__ void k_pair_sum(const uint32_t* in, uint32_t* out, size_t n_out) {
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (i < n_out) out[i] = in[2 * i] + in[2 * i + 1];
}
__global__ void k_slow_fill(uint32_t* out, size_t n) {
  const long long t0 = clock64();
  while (clock64() - t0 < 400000000ll) __nanosleep(1000);  // ~0.2 s at ~2 GHz
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = 41 + uint32_t(i);
}
__global__ void k_add_one(const uint32_t* in, uint32_t* out, size_t n) {
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = in[i] + 1;
}
__global__ void k_times2_inplace(uint32_t* b, size_t n) {
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  if (i < n) b[i] *= 2;
}
__global__ void k_scale_via_local(const float* in, float* out, float s, size_t n) {
  extern __shared__ float loc[];
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  loc[threadIdx.x] = i < n ? in[i] * s : 0.f;
  __syncthreads();
  if (i < n) out[i] = loc[threadIdx.x];
}
__global__ void k_increment(uint32_t* c) {
  if (threadIdx.x == 0) c[0] += 1;
}

static dim3 g3(const LaunchParams& lp) { return dim3(lp.grid[0], lp.grid[1], lp.grid[2]); }
static dim3 b3(const LaunchParams& lp) { return dim3(lp.block[0], lp.block[1], lp.block[2]); }
static int last_err() { return int(cudaGetLastError()); }

#define LAUNCHER(...) [](const LaunchParams& lp) -> int { __VA_ARGS__; return last_err(); }

static KernelDef square_kernel() {
  return KernelDef("square", LAUNCHER(k_square<<<g3(lp), b3(lp), 0, (cudaStream_t)lp.stream>>>(
                                 (const uint32_t*)lp.ptr[0], (uint32_t*)lp.ptr[1], lp.len[1])));
}

static void settle(ActorSystem& sys, Device& dev) {
  sys.await_idle();
  dev.await_all();
}

// ---------------------------------------------------------------- device ----

TEST("cpu", "ndrange: explicit groups validated, default = largest divisor under cap") {
  CHECK_THROWS_AS(resolve_local(NdRange::linear(10, 3), 256), DeviceError);
  CHECK_THROWS_AS(resolve_local(NdRange::linear(512, 512), 256), DeviceError);
  CHECK_THROWS_AS(resolve_local(NdRange::linear(0), 256), DeviceError);
  CHECK_THROWS_AS(resolve_local(NdRange::linear(8, 0), 256), DeviceError);
  CHECK(resolve_local(NdRange::linear(12, 4), 256)[0] == 4);
  CHECK(resolve_local(NdRange::linear(1000), 256)[0] == 250);
  CHECK(resolve_local(NdRange::linear(97), 64)[0] == 1);
  auto g = resolve_local(NdRange::grid2(64, 48), 256);
  CHECK(g[0] == 64 && g[1] == 4);
}

TEST("gpu", "device: zeroed buffers, live count, write-kernel-read round trip") {
  Device dev;
  Buffer a = dev.create_buffer(ElemType::u32, 8);
  CHECK(dev.live_buffers() == 1);
  CHECK(dev.read<uint32_t>(a) == std::vector<uint32_t>(8, 0));
  Buffer b = dev.create_buffer(ElemType::u32, 8);
  Event w = dev.enqueue_write(a, std::vector<uint32_t>{1, 2, 3, 4, 5, 6, 7, 8});
  Event k = dev.enqueue_kernel(square_kernel(), NdRange::linear(8, 8), {KernelArg::global(a), KernelArg::global(b)}, {w});
  CHECK((dev.read<uint32_t>(b, {k}) == std::vector<uint32_t>{1, 4, 9, 16, 25, 36, 49, 64}));
  CHECK_THROWS_AS(dev.enqueue_write(a, std::vector<uint32_t>{1, 2}), DeviceError);
  dev.free_buffer(a);
  dev.free_buffer(b);
  CHECK(dev.live_buffers() == 0);
  CHECK_THROWS_AS(dev.free_buffer(a), DeviceError);
}

TEST("gpu", "device: dependency chains, failure propagation, freed buffers") {
  Device dev;
  Buffer c = dev.create_buffer(ElemType::u32, 1);
  KernelDef inc("increment", LAUNCHER(k_increment<<<1, 32, 0, (cudaStream_t)lp.stream>>>((uint32_t*)lp.ptr[0])));
  Event last;
  for (int i = 0; i < 100; ++i)
    last = dev.enqueue_kernel(inc, NdRange::linear(32, 32), {KernelArg::global(c)}, last.valid() ? std::vector<Event>{last} : std::vector<Event>{});
  CHECK(dev.read<uint32_t>(c, {last})[0] == 100);

  KernelDef bad("bad_launch", [](const LaunchParams&) -> int { return int(cudaErrorInvalidConfiguration); });
  Event f = dev.enqueue_kernel(bad, NdRange::linear(1), {KernelArg::global(c)});
  CHECK(f.await() == EventState::failed);
  CHECK(f.error().find("bad_launch") != std::string::npos);
  Event dep = dev.enqueue_kernel(inc, NdRange::linear(32, 32), {KernelArg::global(c)}, {f});
  CHECK(dep.await() == EventState::failed);
  CHECK(dep.error() == "dependency failed");

  Event inflight = dev.enqueue_kernel(inc, NdRange::linear(32, 32), {KernelArg::global(c)});
  dev.free_buffer(c);
  CHECK(inflight.await() == EventState::complete);
  CHECK_THROWS_AS(dev.enqueue_kernel(inc, NdRange::linear(32, 32), {KernelArg::global(c)}), DeviceError);
  dev.await_all();
  CHECK(dev.live_buffers() == 0);
}

TEST("gpu", "device: callbacks exactly once, host-event dependencies defer the issue") {
  Device dev;
  Buffer c = dev.create_buffer(ElemType::u32, 1);
  KernelDef inc("increment", LAUNCHER(k_increment<<<1, 32, 0, (cudaStream_t)lp.stream>>>((uint32_t*)lp.ptr[0])));
  Event gate = Event::create();
  Event k = dev.enqueue_kernel(inc, NdRange::linear(32, 32), {KernelArg::global(c)}, {gate});
  std::atomic<int> first{0}, second{0};
  k.add_callback([&](EventState) { first.fetch_add(1); });
  std::this_thread::sleep_for(std::chrono::milliseconds(30));
  CHECK(k.state() == EventState::pending);  // waits on the host event
  gate.complete();
  CHECK(k.await() == EventState::complete);
  k.add_callback([&](EventState) { second.fetch_add(1); });  // already terminal: runs now
  dev.await_all();
  CHECK(first.load() == 1);
  CHECK(second.load() == 1);
  CHECK(dev.read<uint32_t>(c)[0] == 1);
  dev.free_buffer(c);
}

TEST("gpu", "memref: shares count, last release frees, drop releases, retrieve waits") {
  Device dev;
  {
    Buffer b = dev.create_buffer(ElemType::u32, 4);
    MemRef r(b, Event{});
    MemRef s = r.share();
    CHECK(r.use_count() == 2);
    r.release();
    CHECK(dev.live_buffers() == 1);
    CHECK_THROWS_AS(r.release(), DeviceError);
    s.release();
    CHECK(dev.live_buffers() == 0);
  }
  {
    Buffer b = dev.create_buffer(ElemType::u32, 4);
    { MemRef dropped(b, Event{}); }
    CHECK(dev.live_buffers() == 0);
  }
  Buffer b = dev.create_buffer(ElemType::u32, 2);
  Event gate = Event::create();
  Event w = dev.enqueue_write(b, std::vector<uint32_t>{7, 9}, {gate});
  MemRef r(b, w);
  std::thread t([&] {
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
    gate.complete();
  });
  CHECK((retrieve_u32(r) == std::vector<uint32_t>{7, 9}));
  t.join();
  r.release();
  dev.await_all();
  CHECK(dev.live_buffers() == 0);
}

// -------------------------------------------------------- compute actor ----

TEST("gpu", "compute: arrays in and out, default out size, SizeFn") {
  ActorSystem sys(2);
  Device dev;
  ComputeActorSpec spec;
  spec.kernel = square_kernel();
  spec.range = NdRange::linear(8);
  spec.args = {ArgSpec::in(ElemType::u32), ArgSpec::out(ElemType::u32)};
  auto sq = spawn_compute(sys, dev, spec);
  Reply r = sys.request(sq, Message::of(std::vector<uint32_t>{1, 2, 3, 4, 5, 6, 7, 8})).await();
  REQUIRE(!is_error(r));
  CHECK((get_message(r).at(0).as_u32s() == std::vector<uint32_t>{1, 4, 9, 16, 25, 36, 49, 64}));

  ComputeActorSpec io;
  io.kernel = KernelDef("iota", LAUNCHER(k_iota<<<g3(lp), b3(lp), 0, (cudaStream_t)lp.stream>>>((uint32_t*)lp.ptr[0], lp.len[0])));
  io.range = NdRange::linear(12);
  io.args = {ArgSpec::out(ElemType::u32)};
  Reply r2 = sys.request(spawn_compute(sys, dev, io), Message{}).await();
  REQUIRE(!is_error(r2));
  CHECK(get_message(r2).at(0).as_u32s().size() == 12);
  CHECK(get_message(r2).at(0).as_u32s()[11] == 11);

  ComputeActorSpec ps;
  ps.kernel = KernelDef("pair_sum", LAUNCHER(k_pair_sum<<<g3(lp), b3(lp), 0, (cudaStream_t)lp.stream>>>(
                                        (const uint32_t*)lp.ptr[0], (uint32_t*)lp.ptr[1], lp.len[1])));
  ps.range_fn = [](const Message& m) { return NdRange::linear(m.at(0).array_length()); };
  ps.args = {ArgSpec::in(ElemType::u32), ArgSpec::out(ElemType::u32, SizeFn{[](const Message& m) { return m.at(0).array_length() / 2; }})};
  Reply r3 = sys.request(spawn_compute(sys, dev, ps), Message::of(std::vector<uint32_t>{1, 2, 3, 4, 5, 6})).await();
  REQUIRE(!is_error(r3));
  CHECK((get_message(r3).at(0).as_u32s() == std::vector<uint32_t>{3, 7, 11}));
  settle(sys, dev);
  CHECK(dev.live_buffers() == 0);
}

TEST("gpu", "compute: mismatch and released-reference errors") {
  ActorSystem sys(2);
  Device dev;
  ComputeActorSpec spec;
  spec.kernel = square_kernel();
  spec.range = NdRange::linear(4);
  spec.args = {ArgSpec::in(ElemType::u32), ArgSpec::out(ElemType::u32)};
  auto sq = spawn_compute(sys, dev, spec);
  Reply wrong = sys.request(sq, Message::of(std::vector<float>{1, 2})).await();
  CHECK(is_error(wrong) && get_error(wrong).code == ErrorCode::mismatch);
  Reply few = sys.request(sq, Message{}).await();
  CHECK(is_error(few) && get_error(few).code == ErrorCode::mismatch);
  Reply many = sys.request(sq, Message::of(std::vector<uint32_t>{1}, std::vector<uint32_t>{2})).await();
  CHECK(is_error(many) && get_error(many).code == ErrorCode::mismatch);

  ComputeActorSpec rs = spec;
  rs.args = {ArgSpec::in(ElemType::u32, ArgMode::ref), ArgSpec::out(ElemType::u32)};
  auto byref = spawn_compute(sys, dev, rs);
  Buffer b = dev.create_buffer(ElemType::u32, 4);
  MemRef ref(b, Event{});
  MemRef keep = ref.share();
  ref.release();
  Reply rel = sys.request(byref, Message::of(ref)).await();
  CHECK(is_error(rel) && get_error(rel).code == ErrorCode::released_ref);
  keep.release();
  settle(sys, dev);
  CHECK(dev.live_buffers() == 0);
}

TEST("gpu", "compute: reference outputs reply before the kernel finishes") {
  ActorSystem sys(2);
  Device dev;
  ComputeActorSpec spec;
  spec.kernel = KernelDef("slow_fill", LAUNCHER(k_slow_fill<<<g3(lp), b3(lp), 0, (cudaStream_t)lp.stream>>>((uint32_t*)lp.ptr[0], lp.len[0])));
  spec.range = NdRange::linear(2, 2);
  spec.args = {ArgSpec::out(ElemType::u32, ArgMode::ref)};
  auto a = spawn_compute(sys, dev, spec);
  auto t0 = Clock::now();
  Reply r = sys.request(a, Message{}).await();
  auto reply_ms = std::chrono::duration_cast<std::chrono::milliseconds>(Clock::now() - t0).count();
  REQUIRE(!is_error(r));
  REQUIRE(get_message(r).at(0).kind() == ValueKind::mem_ref);
  CHECK(reply_ms < 100);
  MemRef out = get_message(r).at(0).as_ref();
  CHECK((retrieve_u32(out) == std::vector<uint32_t>{41, 42}));
  auto total_ms = std::chrono::duration_cast<std::chrono::milliseconds>(Clock::now() - t0).count();
  CHECK(total_ms >= 100);
  out.release();
  settle(sys, dev);
  CHECK(dev.live_buffers() == 0);
}

TEST("gpu", "compute: transfer without a kept share, survival with one") {
  ActorSystem sys(2);
  Device dev;
  ComputeActorSpec spec;
  spec.kernel = KernelDef("sink", LAUNCHER(k_add_one<<<g3(lp), b3(lp), 0, (cudaStream_t)lp.stream>>>(
                                     (const uint32_t*)lp.ptr[0], (uint32_t*)lp.ptr[1], lp.len[1])));
  spec.range = NdRange::linear(4);
  spec.args = {ArgSpec::in(ElemType::u32, ArgMode::ref), ArgSpec::out(ElemType::u32)};
  auto a = spawn_compute(sys, dev, spec);
  Buffer b = dev.create_buffer(ElemType::u32, 4);
  Event w = dev.enqueue_write(b, std::vector<uint32_t>{1, 1, 1, 1});
  {
    MemRef ref(b, w);
    Reply r = sys.request(a, Message::of(ref)).await();
    REQUIRE(!is_error(r));
    CHECK(get_message(r).at(0).as_u32s() == std::vector<uint32_t>(4, 2));
    CHECK(dev.live_buffers() == 1);  // `ref` still holds it
  }
  settle(sys, dev);
  CHECK(dev.live_buffers() == 0);
  Buffer b2 = dev.create_buffer(ElemType::u32, 4);
  MemRef mine(b2, Event{});
  Reply r2 = sys.request(a, Message::of(mine.share())).await();
  REQUIRE(!is_error(r2));
  settle(sys, dev);
  CHECK(dev.live_buffers() == 1);
  mine.release();
  CHECK(dev.live_buffers() == 0);
}

TEST("gpu", "compute: in_out references are forwarded and chain") {
  ActorSystem sys(2);
  Device dev;
  ComputeActorSpec spec;
  spec.kernel = KernelDef("double_in_place", LAUNCHER(k_times2_inplace<<<g3(lp), b3(lp), 0, (cudaStream_t)lp.stream>>>((uint32_t*)lp.ptr[0], lp.len[0])));
  spec.range = NdRange::linear(4);
  spec.args = {ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref)};
  auto a = spawn_compute(sys, dev, spec);
  Buffer b = dev.create_buffer(ElemType::u32, 4);
  Event w = dev.enqueue_write(b, std::vector<uint32_t>{1, 2, 3, 4});
  MemRef ref(b, w);
  const uint64_t id = ref.buffer().id();
  Reply r1 = sys.request(a, Message::of(ref)).await();
  REQUIRE(!is_error(r1));
  MemRef o1 = get_message(r1).at(0).as_ref();
  CHECK(o1.buffer().id() == id);
  Reply r2 = sys.request(a, Message::of(o1)).await();
  MemRef o2 = get_message(r2).at(0).as_ref();
  CHECK((retrieve_u32(o2) == std::vector<uint32_t>{4, 8, 12, 16}));
  o2.release();
  settle(sys, dev);
  CHECK(dev.live_buffers() == 0);
}

TEST("gpu", "compute: priv scalars and local scratch reach the kernel") {
  ActorSystem sys(2);
  Device dev;
  ComputeActorSpec spec;
  spec.kernel = KernelDef("scale_via_local", [](const LaunchParams& lp) -> int {
    k_scale_via_local<<<g3(lp), b3(lp), lp.shared_bytes, (cudaStream_t)lp.stream>>>(
        (const float*)lp.ptr[0], (float*)lp.ptr[1], lp.scalar[3].as<float>(), lp.len[1]);
    return last_err();
  });
  spec.range = NdRange::linear(8, 4);
  spec.args = {ArgSpec::in(ElemType::f32), ArgSpec::out(ElemType::f32), ArgSpec::local(ElemType::f32, 4),
               ArgSpec::priv(Scalar(2.5f))};
  Reply r = sys.request(spawn_compute(sys, dev, spec), Message::of(std::vector<float>{1, 2, 3, 4, 5, 6, 7, 8})).await();
  REQUIRE(!is_error(r));
  CHECK((get_message(r).at(0).as_f32s() == std::vector<float>{2.5f, 5, 7.5f, 10, 12.5f, 15, 17.5f, 20}));
}

TEST("gpu", "compute: preprocess shortcut, postprocess, timing hook") {
  ActorSystem sys(2);
  Device dev;
  std::atomic<int> ran{0}, hooked{0};
  ComputeActorSpec spec;
  spec.kernel = square_kernel();
  spec.range = NdRange::linear(4);
  spec.args = {ArgSpec::in(ElemType::u32), ArgSpec::out(ElemType::u32)};
  spec.preprocess = [&ran](Message& m) -> std::optional<Message> {
    if (m.at(0).as_u32s().empty()) return Message::of(std::vector<uint32_t>{});
    ran.fetch_add(1);
    return std::nullopt;
  };
  spec.postprocess = [](Message m) {
    auto xs = m.at(0).take_u32s();
    xs.push_back(99);
    return Message::of(std::move(xs));
  };
  std::atomic<bool> ordered{true};
  spec.timing = [&](const KernelTiming& t) {
    if (!(t.enqueued <= t.exec_start && t.exec_start <= t.terminal)) ordered = false;
    hooked.fetch_add(1);
  };
  auto a = spawn_compute(sys, dev, spec);
  Reply s = sys.request(a, Message::of(std::vector<uint32_t>{})).await();
  CHECK((get_message(s).at(0).as_u32s() == std::vector<uint32_t>{99}));
  CHECK(ran.load() == 0);
  Reply f = sys.request(a, Message::of(std::vector<uint32_t>{1, 2, 3, 4})).await();
  CHECK((get_message(f).at(0).as_u32s() == std::vector<uint32_t>{1, 4, 9, 16, 99}));
  settle(sys, dev);
  CHECK(hooked.load() == 1);
  CHECK(ordered.load());
}

TEST("gpu", "compute: device failures reply device-failure / fail retrieval") {
  ActorSystem sys(2);
  Device dev;
  ComputeActorSpec spec;
  spec.kernel = KernelDef("oob", [](const LaunchParams&) -> int { return int(cudaErrorInvalidConfiguration); });
  spec.range = NdRange::linear(4);
  spec.args = {ArgSpec::in(ElemType::u32), ArgSpec::out(ElemType::u32)};
  Reply r = sys.request(spawn_compute(sys, dev, spec), Message::of(std::vector<uint32_t>{1, 2, 3, 4})).await();
  REQUIRE(is_error(r));
  CHECK(get_error(r).code == ErrorCode::device_failure);
  CHECK(get_error(r).what.find("oob") != std::string::npos);

  ComputeActorSpec rs;
  rs.kernel = KernelDef("oob_ref", [](const LaunchParams&) -> int { return int(cudaErrorInvalidConfiguration); });
  rs.range = NdRange::linear(4);
  rs.args = {ArgSpec::out(ElemType::u32, ArgMode::ref)};
  Reply r2 = sys.request(spawn_compute(sys, dev, rs), Message{}).await();
  REQUIRE(!is_error(r2));
  MemRef out = get_message(r2).at(0).as_ref();
  CHECK_THROWS_AS(retrieve_u32(out), DeviceError);
  out.release();
  settle(sys, dev);
  CHECK(dev.live_buffers() == 0);
}

TEST("gpu", "compute: compute actors compose over references") {
  ActorSystem sys(4);
  Device dev;
  ComputeActorSpec first;
  // double = copy-then-times2 expressed with the kernels above: in -> out = 2*in
  first.kernel = KernelDef("double", [](const LaunchParams& lp) -> int {
    cudaMemcpyAsync(lp.ptr[1], lp.ptr[0], lp.len[0] * 4, cudaMemcpyDeviceToDevice, (cudaStream_t)lp.stream);
    k_times2_inplace<<<1, 32, 0, (cudaStream_t)lp.stream>>>((uint32_t*)lp.ptr[1], lp.len[1]);
    return last_err();
  });
  first.range = NdRange::linear(6);
  first.args = {ArgSpec::in(ElemType::u32), ArgSpec::out(ElemType::u32, ArgMode::ref)};
  ComputeActorSpec second;
  second.kernel = KernelDef("inc", LAUNCHER(k_add_one<<<1, 32, 0, (cudaStream_t)lp.stream>>>((const uint32_t*)lp.ptr[0], (uint32_t*)lp.ptr[1], lp.len[1])));
  second.range = NdRange::linear(6);
  second.args = {ArgSpec::in(ElemType::u32, ArgMode::ref), ArgSpec::out(ElemType::u32)};
  auto f = spawn_compute(sys, dev, first);
  auto g = spawn_compute(sys, dev, second);
  auto pipeline = g * f;
  Reply r = sys.request(pipeline, Message::of(std::vector<uint32_t>{5, 10, 15, 20, 25, 30})).await();
  REQUIRE(!is_error(r));
  CHECK((get_message(r).at(0).as_u32s() == std::vector<uint32_t>{11, 21, 31, 41, 51, 61}));
  settle(sys, dev);
  CHECK(dev.live_buffers() == 0);
}

// ------------------------------------------------------------ WAH device ----

static std::vector<uint32_t> rand_u32(std::mt19937& rng, size_t n, uint32_t lo, uint32_t hi) {
  std::uniform_int_distribution<uint32_t> pick(lo, hi);
  std::vector<uint32_t> v(n);
  for (auto& x : v) x = pick(rng);
  return v;
}

TEST("gpu", "wah: scan matches the serial oracle around block boundaries") {
  Device dev;
  std::mt19937 rng(8001);
  for (size_t n : {1ul, 2ul, 1023ul, 1024ul, 1025ul, 4096ul, 50000ul, 1048577ul}) {
    auto in = rand_u32(rng, n, 0, 9);
    Buffer b = dev.create_buffer(ElemType::u32, int64_t(n));
    Event w = dev.enqueue_write(b, in);
    wah::ScanResult r = wah::scan_exclusive(dev, b, n, {w});
    std::vector<uint32_t> want(n);
    std::exclusive_scan(in.begin(), in.end(), want.begin(), 0u);
    CHECK(dev.read<uint32_t>(r.sums, {r.done}) == want);
    dev.free_buffer(b);
    dev.free_buffer(r.sums);
  }
  CHECK_THROWS_AS(wah::scan_exclusive(dev, dev.create_buffer(ElemType::u32, 1), 0), DeviceError);
  dev.await_all();
}

TEST("gpu", "wah: sort_pairs is stable for every digit width") {
  Device dev;
  std::mt19937 rng(8002);
  for (unsigned bits : {4u, 8u, 16u}) {
    for (size_t n : {1ul, 7ul, 16384ul, 16385ul, 40000ul}) {
      auto keys = rand_u32(rng, n, 0, 5);
      if (n > 20) {
        keys[3] = 0xffffffffu;
        keys[n / 2] = 0x80000000u;
      }
      std::vector<uint32_t> pos(n);
      std::iota(pos.begin(), pos.end(), 0u);
      Buffer kb = dev.create_buffer(ElemType::u32, int64_t(n)), pb = dev.create_buffer(ElemType::u32, int64_t(n));
      Event done = wah::sort_pairs(dev, kb, pb, n, bits, {dev.enqueue_write(kb, keys), dev.enqueue_write(pb, pos)});
      std::vector<uint32_t> want = pos;
      std::stable_sort(want.begin(), want.end(), [&](uint32_t a, uint32_t b) { return keys[a] < keys[b]; });
      std::vector<uint32_t> wk(n);
      for (size_t i = 0; i < n; ++i) wk[i] = keys[want[i]];
      CHECK(dev.read<uint32_t>(kb, {done}) == wk);
      CHECK(dev.read<uint32_t>(pb, {done}) == want);
      dev.free_buffer(kb);
      dev.free_buffer(pb);
    }
  }
  Buffer kb = dev.create_buffer(ElemType::u32, 4);
  CHECK_THROWS_AS(wah::sort_pairs(dev, kb, kb, 4, 5), DeviceError);
  dev.await_all();
}

TEST("gpu", "wah: compaction drops zeros, fused == stepwise") {
  Device dev;
  ActorSystem sys;
  auto st = wah::spawn_compaction(sys, dev);
  std::mt19937 rng(8003);
  for (int it = 0; it < 60; ++it) {
    size_t n = 1 + rng() % 20000;
    std::vector<uint32_t> in = it % 10 == 8 ? std::vector<uint32_t>(n, 0)
                               : it % 10 == 9 ? rand_u32(rng, n, 1, 99)
                                              : rand_u32(rng, n, 0, 2);
    std::vector<uint32_t> want;
    for (uint32_t v : in)
      if (v) want.push_back(v);
    CHECK(wah::compact(sys, dev, st, in) == want);
  }
  for (int it = 0; it < 10; ++it) {
    size_t k = 1 + rng() % 5000;
    auto a = rand_u32(rng, k, 0, 3), b = rand_u32(rng, k, 0, 3);
    auto input = [&] {
      Buffer cfg = dev.create_buffer(ElemType::u32, 2), ab = dev.create_buffer(ElemType::u32, int64_t(k)),
             bb = dev.create_buffer(ElemType::u32, int64_t(k));
      return Message::of(MemRef(cfg, dev.enqueue_write(cfg, std::vector<uint32_t>{uint32_t(k), 0})),
                         MemRef(ab, dev.enqueue_write(ab, a)), MemRef(bb, dev.enqueue_write(bb, b)));
    };
    auto unpack = [](const Reply& r) {
      MemRef c = get_message(r).at(0).as_ref(), d = get_message(r).at(1).as_ref();
      auto cv = retrieve_u32(c);
      auto dv = retrieve_u32(d);
      release(c);
      release(d);
      dv.resize(cv[1]);
      return dv;
    };
    Reply fused = sys.request(st.fused, input()).await();
    REQUIRE(!is_error(fused));
    Reply prep = sys.request(st.prepare, input()).await();
    Reply cnt = sys.request(st.count, get_message(prep)).await();
    Reply mov = sys.request(st.move, get_message(cnt)).await();
    REQUIRE(!is_error(mov));
    CHECK(unpack(fused) == unpack(mov));
  }
  settle(sys, dev);
  CHECK(dev.live_buffers() == 0);
}

TEST("gpu", "wah: build_index equals the reference word for word") {
  Device dev;
  ActorSystem sys;
  std::mt19937 rng(8005);
  const uint32_t cards[] = {1, 2, 10, 1000};
  for (int it = 0; it < 24; ++it) {
    size_t n = 1 + rng() % 30000;
    auto v = rand_u32(rng, n, 0, cards[it % 4] - 1);
    for (auto& x : v) x = x * 37 + 11;
    REQUIRE(wah::build_index(sys, dev, v) == oracle_index(v));
  }
  std::vector<uint32_t> clustered;
  for (int b = 0; b < 200; ++b) clustered.insert(clustered.end(), 150, uint32_t(b % 3));
  wah::WahIndex ci = wah::build_index(sys, dev, clustered);
  CHECK(ci == oracle_index(clustered));
  CHECK(std::any_of(ci.words.begin(), ci.words.end(), wah::is_ones_fill));
  wah::WahIndex one = wah::build_index(sys, dev, std::vector<uint32_t>{77});
  CHECK(one.words == std::vector<uint32_t>{1});
  wah::WahIndex none = wah::build_index(sys, dev, std::vector<uint32_t>{});
  CHECK(none.row_count == 0 && none.entries.empty() && none.words.empty());
  auto v = rand_u32(rng, 9000, 0, 40);
  wah::WahIndex wide = wah::build_index(sys, dev, v, 16);
  CHECK(wah::build_index(sys, dev, v, 8) == wide);
  CHECK(wah::build_index(sys, dev, v, 4) == wide);
  // rows_for recovers positions from the device-built index
  for (uint32_t q : {0u, 7u, 40u}) {
    std::vector<uint32_t> want;
    for (uint32_t r = 0; r < v.size(); ++r)
      if (v[r] == q) want.push_back(r);
    CHECK(wah::rows_for(wide, q) == want);
  }
  settle(sys, dev);
  CHECK(dev.live_buffers() == 0);
}

TEST("gpu", "wah: index file round trip of a device-built index") {
  Device dev;
  ActorSystem sys;
  std::mt19937 rng(5);
  std::uniform_int_distribution<uint32_t> pick(0, 6);  // test_cli.cpp:61-80 shape
  std::vector<uint32_t> v(3000);
  for (auto& x : v) x = pick(rng);
  wah::WahIndex idx = wah::build_index(sys, dev, v);
  CHECK(wah::serialize_index(idx) == wah::serialize_index(oracle_index(v)));
  const std::string path = "/tmp/ndactor_cli_index.wah";
  wah::write_index_file(path, idx);
  CHECK(wah::read_index_file(path) == idx);
}

TEST("gpu", "multi-device: copy_to moves references between devices; foreign refs are a mismatch") {
  // two Devices (own streams, own actors); on a one-GPU box both use ordinal 0
  int count = 0;
  cudaGetDeviceCount(&count);
  ActorSystem sys(2);
  Device a(DeviceConfig{0}), b(DeviceConfig{count > 1 ? 1 : 0});
  ComputeActorSpec spec;
  spec.kernel = KernelDef("double_in_place", LAUNCHER(k_times2_inplace<<<g3(lp), b3(lp), 0, (cudaStream_t)lp.stream>>>((uint32_t*)lp.ptr[0], lp.len[0])));
  spec.range = NdRange::linear(4);
  spec.args = {ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref)};
  auto on_a = spawn_compute(sys, a, spec);
  auto on_b = spawn_compute(sys, b, spec);
  Buffer buf = a.create_buffer(ElemType::u32, 4);
  MemRef ref(buf, a.enqueue_write(buf, std::vector<uint32_t>{1, 2, 3, 4}));
  Reply r1 = sys.request(on_a, Message::of(ref)).await();
  REQUIRE(!is_error(r1));
  MemRef ra = get_message(r1).at(0).as_ref();
  // a reference of device a is not accepted by an actor on device b
  Reply bad = sys.request(on_b, Message::of(ra)).await();
  REQUIRE(is_error(bad));
  CHECK(get_error(bad).code == ErrorCode::mismatch);
  MemRef rb = copy_to(ra, b);
  CHECK(&rb.buffer().device() == &b);
  Reply r2 = sys.request(on_b, Message::of(rb)).await();
  REQUIRE(!is_error(r2));
  CHECK((retrieve_u32(get_message(r2).at(0).as_ref()) == std::vector<uint32_t>{4, 8, 12, 16}));
  CHECK((retrieve_u32(ra) == std::vector<uint32_t>{2, 4, 6, 8}));  // the source is untouched
  get_message(r2).at(0).as_ref().release();
  ra.release();
  settle(sys, a);
  settle(sys, b);
  CHECK(a.live_buffers() == 0);
  CHECK(b.live_buffers() == 0);
}
