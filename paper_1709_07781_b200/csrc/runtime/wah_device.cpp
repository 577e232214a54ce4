// The WAH device API (reference: p/core/include/ndactor/wah_device.hpp:17-58)
// on the B200 kernels of libndx.so, driven through compute actors.
//
//   scan_exclusive / sort_pairs      one native command each
//   spawn_compaction / compact       the paper's Listing 5 actors, same protocol
//                                    (wah_stages.cpp:29-201)
//   spawn_index_stages / build_index the four-stage build chain
//                                    table * emit * sort * plan, every hand-off
//                                    a device-resident MemRef, the counts in a
//                                    device `cfg` block (no host round trip)
#include "ndactor/wah_device.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>

#include "device_impl.hpp"
#include "ndx.h"

namespace ndactor::wah {

namespace {

std::size_t ref_len(const Message& m, std::size_t slot) {
  if (slot >= m.size() || m.at(slot).kind() != ValueKind::mem_ref) return 0;
  return m.at(slot).as_ref().length();
}

NdRange padded_linear(std::size_t n, std::size_t group) {
  const std::size_t groups = (std::max<std::size_t>(n, 1) + group - 1) / group;
  return NdRange::linear(groups * group, group);
}

constexpr std::size_t kStageTile = 4096;  // counts per 4096 elements (wah_stages.cpp:11)
std::size_t stage_groups(std::size_t n) { return (std::max<std::size_t>(n, 1) + kStageTile - 1) / kStageTile; }

// Scratch a launcher needs for one launch: stream-ordered pool allocation,
// freed in stream order right after the kernels that use it.
struct StreamScratch {
  void* p = nullptr;
  void* stream;
  StreamScratch(std::size_t bytes, void* s, bool zero) : stream(s) {
    if (ndx_malloc_async(&p, bytes, s) == 0 && zero) ndx_memset_async(p, 0, bytes, s);
  }
  ~StreamScratch() {
    if (p) ndx_free_async(p, stream);
  }
};

// Per-device build workspace: the look-back status buffer (zeroed once,
// epoch-tagged afterwards), the sort's ping-pong pairs and the emit scratch.
struct Workspace {
  std::mutex mu;
  std::uint64_t cap = 0;
  void* status = nullptr;
  void* tmp_pairs = nullptr;
  void* emit = nullptr;
  void* stream = nullptr;

  void ensure(std::uint64_t n, void* s) {
    std::lock_guard<std::mutex> l(mu);
    if (n <= cap && stream == s) return;
    release_locked();
    stream = s;
    cap = std::max<std::uint64_t>(n, 1 << 16);
    const std::size_t sb = ndx_wah_status_bytes(cap);
    ndx_malloc_async(&status, sb, s);
    ndx_memset_async(status, 0, sb, s);
    ndx_malloc_async(&tmp_pairs, std::size_t(cap) * 8, s);
    ndx_malloc_async(&emit, ndx_wah_emit_scratch_bytes(cap), s);
  }
  void release_locked() {
    if (!stream) return;
    ndx_free_async(status, stream);
    ndx_free_async(tmp_pairs, stream);
    ndx_free_async(emit, stream);
    status = tmp_pairs = emit = nullptr;
  }
  ~Workspace() {
    std::lock_guard<std::mutex> l(mu);
    release_locked();
  }
};

std::mutex g_ws_mu;
std::map<const detail::DeviceImpl*, std::weak_ptr<Workspace>> g_ws;

std::shared_ptr<Workspace> workspace_for(Device& dev) {
  std::lock_guard<std::mutex> l(g_ws_mu);
  auto& w = g_ws[&dev.impl()];
  if (auto s = w.lock()) return s;
  auto s = std::make_shared<Workspace>();
  w = s;
  return s;
}

}  // namespace

// ------------------------------------------------------ primitives ------

ScanResult scan_exclusive(Device& dev, const Buffer& in, std::size_t n, std::vector<Event> deps) {
  if (n == 0) throw DeviceError("scan over an empty range");
  if (n > in.length()) throw DeviceError("scan range exceeds the buffer");
  Buffer out = dev.create_buffer_uninit(ElemType::u32, std::int64_t(n));
  const std::uint32_t* src = static_cast<const std::uint32_t*>(in.data());
  std::uint32_t* dst = static_cast<std::uint32_t*>(out.data());
  Event done = dev.enqueue_native(
      "scan_exclusive",
      [src, dst, n](void* s) -> int {
        StreamScratch scr(ndx_scan_scratch_bytes(n), s, false);
        return ndx_scan_exclusive_u32(src, dst, n, scr.p, s);
      },
      std::move(deps));
  return {out, done};
}

Event sort_pairs(Device& dev, const Buffer& keys, const Buffer& payloads, std::size_t n,
                 unsigned digit_bits, std::vector<Event> deps) {
  if (digit_bits != 4 && digit_bits != 8 && digit_bits != 16)
    throw DeviceError("digit width must be 4, 8, or 16 bits");
  if (n == 0) throw DeviceError("sort over an empty range");
  if (n > keys.length() || n > payloads.length()) throw DeviceError("sort range exceeds the buffers");
  auto* k = static_cast<std::uint32_t*>(keys.data());
  auto* p = static_cast<std::uint32_t*>(payloads.data());
  return dev.enqueue_native(
      "sort_pairs",
      [k, p, n](void* s) -> int {
        StreamScratch scr(ndx_sort_pairs_scratch_bytes(n), s, false);
        return ndx_sort_pairs_u32(k, p, n, scr.p, s);
      },
      std::move(deps));
}

// ------------------------------------------------------ compaction ------

CompactionStages spawn_compaction(ActorSystem& sys, Device& dev) {
  const std::size_t group = 128;

  // prepare: (config, a, b) -> (config, a0 b0 a1 b1 ...)        wah_stages.cpp:33-57
  ComputeActorSpec prepare;
  prepare.kernel = KernelDef("compact_prepare", [](const LaunchParams& lp) -> int {
    return ndx_compact_prepare(static_cast<std::uint32_t*>(lp.ptr[0]),
                               static_cast<const std::uint32_t*>(lp.ptr[1]),
                               static_cast<const std::uint32_t*>(lp.ptr[2]), lp.len[1],
                               static_cast<std::uint32_t*>(lp.ptr[3]), lp.stream);
  });
  prepare.args = {ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref),
                  ArgSpec::in(ElemType::u32, ArgMode::ref), ArgSpec::in(ElemType::u32, ArgMode::ref),
                  ArgSpec::out(ElemType::u32, SizeFn{[](const Message& m) { return 2 * ref_len(m, 1); }},
                               ArgMode::ref)
                      .uninitialized()};
  prepare.range_fn = [group](const Message& m) { return padded_linear(ref_len(m, 1), group); };

  // count: (config, data) -> (config, data, per-tile nonzero counts)  wah_stages.cpp:59-91
  ComputeActorSpec count;
  count.kernel = KernelDef("compact_count", [](const LaunchParams& lp) -> int {
    return ndx_compact_count(static_cast<const std::uint32_t*>(lp.ptr[1]), lp.len[1],
                             static_cast<std::uint32_t*>(lp.ptr[2]), lp.stream);
  });
  count.args = {ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref),
                ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref),
                ArgSpec::out(ElemType::u32, SizeFn{[](const Message& m) { return stage_groups(ref_len(m, 1)); }},
                             ArgMode::ref)
                    .uninitialized(),
                ArgSpec::local(ElemType::u32, group)};
  count.range_fn = [group](const Message& m) {
    return NdRange::linear(stage_groups(ref_len(m, 1)) * group, group);
  };

  // move: (config, data, counts) -> (config, compacted); config[1] = total  wah_stages.cpp:93-156
  ComputeActorSpec move;
  move.kernel = KernelDef("compact_move", [](const LaunchParams& lp) -> int {
    const std::size_t n = lp.len[1];
    StreamScratch scr(ndx_compact_move_scratch_bytes(n), lp.stream, false);
    return ndx_compact_move(static_cast<std::uint32_t*>(lp.ptr[0]),
                            static_cast<const std::uint32_t*>(lp.ptr[1]), n,
                            static_cast<const std::uint32_t*>(lp.ptr[2]),
                            static_cast<std::uint32_t*>(lp.ptr[3]), scr.p, lp.stream);
  });
  move.args = {ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref),
               ArgSpec::in(ElemType::u32, ArgMode::ref), ArgSpec::in(ElemType::u32, ArgMode::ref),
               ArgSpec::out(ElemType::u32, SizeFn{[](const Message& m) { return ref_len(m, 1); }}, ArgMode::ref),
               ArgSpec::local(ElemType::u32, group), ArgSpec::local(ElemType::u32, 1)};
  move.range_fn = [group](const Message& m) {
    return NdRange::linear(stage_groups(ref_len(m, 1)) * group, group);
  };

  CompactionStages st;
  st.prepare = spawn_compute(sys, dev, std::move(prepare));
  st.count = spawn_compute(sys, dev, std::move(count));
  st.move = spawn_compute(sys, dev, std::move(move));
  st.fused = sys.compose(st.move, sys.compose(st.count, st.prepare));
  return st;
}

std::vector<std::uint32_t> compact(ActorSystem& sys, Device& dev, const CompactionStages& stages,
                                   std::span<const std::uint32_t> input) {
  if (input.empty()) return {};
  // prepare reassembles a0 b0 a1 b1 ...: feed it the even and odd positions
  const std::size_t k = (input.size() + 1) / 2;
  std::vector<std::uint32_t> a(k, 0), b(k, 0);
  for (std::size_t i = 0; i < input.size(); ++i) (i % 2 ? b : a)[i / 2] = input[i];
  Buffer cfg = dev.create_buffer(ElemType::u32, 2);
  Buffer ab = dev.create_buffer_uninit(ElemType::u32, std::int64_t(k));
  Buffer bb = dev.create_buffer_uninit(ElemType::u32, std::int64_t(k));
  Event wc = dev.enqueue_write(cfg, std::vector<std::uint32_t>{std::uint32_t(k), 0});
  Event wa = dev.enqueue_write(ab, a);
  Event wb = dev.enqueue_write(bb, b);
  Reply r = sys.request(stages.fused, Message::of(MemRef(cfg, wc), MemRef(ab, wa), MemRef(bb, wb))).await();
  if (is_error(r)) throw DeviceError("compaction failed: " + get_error(r).what);
  const Message& m = get_message(r);
  MemRef cfg_back = m.at(0).as_ref();
  MemRef packed = m.at(1).as_ref();
  const std::uint32_t total = retrieve_u32(cfg_back)[1];
  std::vector<std::uint32_t> words = retrieve_u32(packed);
  release(cfg_back);
  release(packed);
  words.resize(total);
  return words;
}

// ------------------------------------------------------ index chain -----

IndexStages spawn_index_stages(ActorSystem& sys, Device& dev, std::uint32_t row_base) {
  auto ws = workspace_for(dev);
  const std::size_t ctl_words = ndx_wah_ctl_bytes() / 4;
  const NdRange one = NdRange::linear(1, 1);  // the launchers size their own grids

  // plan: {keys} -> {cfg, keys}
  ComputeActorSpec plan;
  plan.kernel = KernelDef("wah_plan", [ws](const LaunchParams& lp) -> int {
    const std::uint64_t n = lp.len[1];
    if (n == 0) return 0;
    ws->ensure(n, lp.stream);
    return ndx_wah_plan(static_cast<const std::uint32_t*>(lp.ptr[1]), n, lp.ptr[0], ws->status, lp.stream);
  });
  plan.args = {ArgSpec::out(ElemType::u32, ctl_words, ArgMode::ref),
               ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref)};
  plan.range = one;

  // sort: {cfg, keys} -> {cfg, pairs}
  ComputeActorSpec sort;
  sort.kernel = KernelDef("wah_sort", [ws, row_base](const LaunchParams& lp) -> int {
    const std::uint64_t n = lp.len[1];
    if (n == 0) return 0;
    ws->ensure(n, lp.stream);
    return ndx_wah_sort(static_cast<const std::uint32_t*>(lp.ptr[1]), n, row_base, lp.ptr[0],
                        static_cast<std::uint64_t*>(lp.ptr[2]),
                        static_cast<std::uint64_t*>(ws->tmp_pairs), ws->status, lp.stream);
  });
  sort.args = {ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref),
               ArgSpec::in(ElemType::u32, ArgMode::ref),
               ArgSpec::out(ElemType::u32, SizeFn{[](const Message& m) { return 2 * ref_len(m, 1); }},
                            ArgMode::ref)
                   .uninitialized()};
  sort.range = one;

  // emit: {cfg, pairs} -> {cfg, words, vstart, values}
  ComputeActorSpec emit;
  emit.kernel = KernelDef("wah_emit", [ws](const LaunchParams& lp) -> int {
    const std::uint64_t n = lp.len[1] / 2;
    if (n == 0) return 0;
    ws->ensure(n, lp.stream);
    return ndx_wah_emit(static_cast<const std::uint64_t*>(lp.ptr[1]), n, lp.ptr[0],
                        static_cast<std::uint32_t*>(lp.ptr[2]), static_cast<std::uint32_t*>(lp.ptr[3]),
                        static_cast<std::uint32_t*>(lp.ptr[4]), ws->emit, lp.stream);
  });
  auto n_of_pairs = [](const Message& m) { return ref_len(m, 1) / 2; };
  emit.args = {ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref),
               ArgSpec::in(ElemType::u32, ArgMode::ref),
               ArgSpec::out(ElemType::u32, SizeFn{[=](const Message& m) { return 2 * n_of_pairs(m); }},
                            ArgMode::ref)
                   .uninitialized(),
               ArgSpec::out(ElemType::u32, SizeFn{n_of_pairs}, ArgMode::ref).uninitialized(),
               ArgSpec::out(ElemType::u32, SizeFn{n_of_pairs}, ArgMode::ref).uninitialized()};
  emit.range = one;

  // table: {cfg, words, vstart, values} -> {cfg, words, entries}
  ComputeActorSpec table;
  table.kernel = KernelDef("wah_table", [](const LaunchParams& lp) -> int {
    const std::uint64_t n = lp.len[2];
    return ndx_wah_table(static_cast<const std::uint32_t*>(lp.ptr[3]),
                         static_cast<const std::uint32_t*>(lp.ptr[2]), n, lp.ptr[0],
                         static_cast<std::uint32_t*>(lp.ptr[4]), lp.stream);
  });
  table.args = {ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref),
                ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref),
                ArgSpec::in(ElemType::u32, ArgMode::ref), ArgSpec::in(ElemType::u32, ArgMode::ref),
                ArgSpec::out(ElemType::u32, SizeFn{[](const Message& m) { return 3 * ref_len(m, 2); }},
                             ArgMode::ref)
                    .uninitialized()};
  table.range = one;

  IndexStages st;
  st.plan = spawn_compute(sys, dev, std::move(plan));
  st.sort = spawn_compute(sys, dev, std::move(sort));
  st.emit = spawn_compute(sys, dev, std::move(emit));
  st.table = spawn_compute(sys, dev, std::move(table));
  st.chain = st.table * st.emit * st.sort * st.plan;
  return st;
}

// ------------------------------------------------------ shard chain -----
//
// The multi-GPU build's local chain: the same plan, sort, emit and table
// kernels with the shard's global row base, but
//   * the words land in a caller buffer that travels with the message (a
//     cudaMalloc'd buffer other GPUs map over NVLink), and
//   * the sorted pairs travel on to a fifth stage, the shard metadata
//     (ndx_wah_shard_meta_dev: per value its first/last chunk and end fills,
//     at most meta_cap records, the count read on the device).
// {keys, wbuf} -> plan -> sort -> emit -> table -> meta -> {cfg, wbuf, entries, meta}

ShardStages spawn_shard_stages(ActorSystem& sys, Device& dev, std::uint32_t row_base, std::uint32_t meta_cap) {
  auto ws = workspace_for(dev);
  const std::size_t ctl_words = ndx_wah_ctl_bytes() / 4;
  const NdRange one = NdRange::linear(1, 1);
  const ArgSpec fwd = ArgSpec::in_out(ElemType::u32, ArgMode::ref, ArgMode::ref);

  // plan: {keys, wbuf} -> {cfg, keys, wbuf}
  ComputeActorSpec plan;
  plan.kernel = KernelDef("wah_plan", [ws](const LaunchParams& lp) -> int {
    const std::uint64_t n = lp.len[1];
    if (n == 0) return 0;
    ws->ensure(n, lp.stream);
    return ndx_wah_plan(static_cast<const std::uint32_t*>(lp.ptr[1]), n, lp.ptr[0], ws->status, lp.stream);
  });
  plan.args = {ArgSpec::out(ElemType::u32, ctl_words, ArgMode::ref), fwd, fwd};
  plan.range = one;

  // sort: {cfg, keys, wbuf} -> {cfg, pairs, wbuf}
  ComputeActorSpec sort;
  sort.kernel = KernelDef("wah_sort", [ws, row_base](const LaunchParams& lp) -> int {
    const std::uint64_t n = lp.len[1];
    if (n == 0) return 0;
    ws->ensure(n, lp.stream);
    return ndx_wah_sort(static_cast<const std::uint32_t*>(lp.ptr[1]), n, row_base, lp.ptr[0],
                        static_cast<std::uint64_t*>(lp.ptr[2]), static_cast<std::uint64_t*>(ws->tmp_pairs),
                        ws->status, lp.stream);
  });
  sort.args = {fwd, ArgSpec::in(ElemType::u32, ArgMode::ref),
               ArgSpec::out(ElemType::u32, SizeFn{[](const Message& m) { return 2 * ref_len(m, 1); }},
                            ArgMode::ref)
                   .uninitialized(),
               fwd};
  sort.range = one;

  // emit: {cfg, pairs, wbuf} -> {cfg, pairs, wbuf, vstart, values}
  ComputeActorSpec emit;
  emit.kernel = KernelDef("wah_emit", [ws](const LaunchParams& lp) -> int {
    const std::uint64_t n = lp.len[1] / 2;
    if (n == 0) return 0;
    if (lp.len[2] < 2 * n) return NDX_E_INVALID;  // the word buffer holds at most 2 words per value
    ws->ensure(n, lp.stream);
    return ndx_wah_emit(static_cast<const std::uint64_t*>(lp.ptr[1]), n, lp.ptr[0],
                        static_cast<std::uint32_t*>(lp.ptr[2]), static_cast<std::uint32_t*>(lp.ptr[3]),
                        static_cast<std::uint32_t*>(lp.ptr[4]), ws->emit, lp.stream);
  });
  auto n_of_pairs = [](const Message& m) { return ref_len(m, 1) / 2; };
  emit.args = {fwd, fwd, fwd, ArgSpec::out(ElemType::u32, SizeFn{n_of_pairs}, ArgMode::ref).uninitialized(),
               ArgSpec::out(ElemType::u32, SizeFn{n_of_pairs}, ArgMode::ref).uninitialized()};
  emit.range = one;

  // table: {cfg, pairs, wbuf, vstart, values} -> {cfg, pairs, wbuf, entries}
  ComputeActorSpec table;
  table.kernel = KernelDef("wah_table", [](const LaunchParams& lp) -> int {
    const std::uint64_t n = lp.len[3];
    return ndx_wah_table(static_cast<const std::uint32_t*>(lp.ptr[4]),
                         static_cast<const std::uint32_t*>(lp.ptr[3]), n, lp.ptr[0],
                         static_cast<std::uint32_t*>(lp.ptr[5]), lp.stream);
  });
  table.args = {fwd, fwd, fwd, ArgSpec::in(ElemType::u32, ArgMode::ref), ArgSpec::in(ElemType::u32, ArgMode::ref),
                ArgSpec::out(ElemType::u32, SizeFn{[](const Message& m) { return 3 * ref_len(m, 3); }},
                             ArgMode::ref)
                    .uninitialized()};
  table.range = one;

  // meta: {cfg, pairs, wbuf, entries} -> {cfg, wbuf, entries, meta}
  ComputeActorSpec meta;
  meta.kernel = KernelDef("wah_shard_meta", [meta_cap](const LaunchParams& lp) -> int {
    const std::uint64_t n = lp.len[1] / 2;
    if (n == 0) return 0;
    return ndx_wah_shard_meta_dev(static_cast<const std::uint64_t*>(lp.ptr[1]), n,
                                  static_cast<const std::uint32_t*>(lp.ptr[3]), lp.ptr[0], meta_cap,
                                  static_cast<const std::uint32_t*>(lp.ptr[2]),
                                  static_cast<ndx_shard_meta*>(lp.ptr[4]), lp.stream);
  });
  meta.args = {fwd, ArgSpec::in(ElemType::u32, ArgMode::ref), fwd, fwd,
               ArgSpec::out(ElemType::u32, std::size_t(meta_cap) * (sizeof(ndx_shard_meta) / 4), ArgMode::ref)
                   .uninitialized()};
  meta.range = one;

  ShardStages st;
  st.plan = spawn_compute(sys, dev, std::move(plan));
  st.sort = spawn_compute(sys, dev, std::move(sort));
  st.emit = spawn_compute(sys, dev, std::move(emit));
  st.table = spawn_compute(sys, dev, std::move(table));
  st.meta = spawn_compute(sys, dev, std::move(meta));
  st.chain = st.meta * st.table * st.emit * st.sort * st.plan;
  return st;
}

DeviceIndex build_index_device(ActorSystem& sys, const IndexStages& stages, MemRef keys,
                               std::uint32_t row_count) {
  Reply r = sys.request(stages.chain, Message::of(std::move(keys))).await();
  if (is_error(r)) throw WahError("index build failed: " + get_error(r).what);
  const Message& m = get_message(r);
  DeviceIndex d;
  d.row_count = row_count;
  d.cfg = m.at(0).as_ref();
  d.words = m.at(1).as_ref();
  d.entries = m.at(2).as_ref();
  return d;
}

WahIndex fetch_index(const DeviceIndex& d) {
  WahIndex idx;
  idx.row_count = d.row_count;
  if (!d.cfg.valid()) return idx;
  // counts first (24 bytes), then exactly W words and D entries
  Buffer cfg = d.cfg.buffer();
  Device& dev = cfg.device();
  std::vector<Event> deps;
  if (d.entries.pending().valid()) deps.push_back(d.entries.pending());
  ndx_wah_counts counts{};
  Event got = dev.enqueue_native(
      "fetch_counts",
      [&counts, p = cfg.data()](void* s) { return ndx_memcpy_d2h_async(&counts, p, sizeof(counts), s); },
      deps);
  if (got.await() == EventState::failed) throw WahError("index build failed: " + got.error());
  idx.words.resize(counts.words);
  std::vector<std::uint32_t> ent(3 * counts.distinct);
  Event rd = dev.enqueue_native(
      "fetch_index",
      [&, pw = d.words.buffer().data(), pe = d.entries.buffer().data()](void* s) -> int {
        int rc = ndx_memcpy_d2h_async(idx.words.data(), pw, idx.words.size() * 4, s);
        if (!rc) rc = ndx_memcpy_d2h_async(ent.data(), pe, ent.size() * 4, s);
        return rc;
      },
      {});
  if (rd.await() == EventState::failed) throw WahError("index read-back failed: " + rd.error());
  idx.entries.resize(counts.distinct);
  for (std::size_t i = 0; i < idx.entries.size(); ++i)
    idx.entries[i] = IndexEntry{ent[3 * i], ent[3 * i + 1], ent[3 * i + 2]};
  if (!idx.entries.empty() && std::uint64_t(idx.entries.back().offset) + idx.entries.back().length != counts.words)
    throw WahError("pipeline produced inconsistent word offsets");
  return idx;
}

WahIndex build_index(ActorSystem& sys, Device& dev, std::span<const std::uint32_t> values,
                     unsigned digit_bits) {
  if (digit_bits != 4 && digit_bits != 8 && digit_bits != 16)
    throw DeviceError("digit width must be 4, 8, or 16 bits");
  WahIndex empty;
  empty.row_count = std::uint32_t(values.size());
  if (values.empty()) return empty;
  if (values.size() >= (std::size_t(1) << 31)) throw WahError("more rows than the u32 index format holds");
  IndexStages stages = spawn_index_stages(sys, dev);
  Buffer keys = dev.create_buffer_uninit(ElemType::u32, std::int64_t(values.size()));
  std::vector<std::byte> bytes(values.size() * 4);
  std::memcpy(bytes.data(), values.data(), bytes.size());
  Event wrote = dev.enqueue_write_bytes(keys, std::move(bytes));
  DeviceIndex d = build_index_device(sys, stages, MemRef(keys, wrote), std::uint32_t(values.size()));
  WahIndex idx = fetch_index(d);
  release(d.cfg);
  release(d.words);
  release(d.entries);
  for (const ActorHandle& a : {stages.chain, stages.table, stages.emit, stages.sort, stages.plan})
    sys.terminate(a);
  return idx;
}

}  // namespace ndactor::wah
