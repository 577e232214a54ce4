// ndactor/wah_device.hpp -- the WAH build on the device.
//
// The reference's public device API (p/core/include/ndactor/wah_device.hpp:
// 10-58) with the same signatures, plus the B200 four-stage build chain.
#pragma once

#include <span>

#include "ndactor/compute_actor.hpp"
#include "ndactor/wah.hpp"

namespace ndactor::wah {

struct ScanResult {
  Buffer sums;
  Event done;
};

/// Exclusive prefix sum (mod 2^32) over the first `n` u32 of `in`
/// (wah_scan.cpp:14-95); single-pass decoupled look-back on the device.
ScanResult scan_exclusive(Device& dev, const Buffer& in, std::size_t n,
                          std::vector<Event> deps = {});

/// Stable sort of (key, payload) pairs by key, in place (wah_radix.cpp:16-127).
/// `digit_bits` must be 4, 8 or 16 as in the reference; the device picks its
/// own digit plan (the result is identical for every digit width).
Event sort_pairs(Device& dev, const Buffer& keys, const Buffer& payloads, std::size_t n,
                 unsigned digit_bits = 16, std::vector<Event> deps = {});

/// The three compaction stages of the paper's Listing 5 (wah_stages.cpp:
/// 29-163), same message protocol: config u32[2] travels by reference,
/// config[0] = k in, config[1] = compacted length out.
struct CompactionStages {
  ActorHandle prepare;
  ActorHandle count;
  ActorHandle move;
  ActorHandle fused;  // move * (count * prepare)
};

CompactionStages spawn_compaction(ActorSystem& sys, Device& dev);

/// Order-preserving removal of zeros through `fused` (wah_stages.cpp:166-201).
std::vector<std::uint32_t> compact(ActorSystem& sys, Device& dev, const CompactionStages& stages,
                                   std::span<const std::uint32_t> input);

/// The B200 build as four compute actors chained by device-resident MemRefs
/// (SURVEY.md section 7 step 6).  Message protocol, all slots MemRefs:
///   plan   {keys u32[n]}                    -> {cfg, keys}
///   sort   {cfg, keys}                      -> {cfg, pairs u32[2n]}
///   emit   {cfg, pairs}                     -> {cfg, words u32[2n], vstart, values}
///   table  {cfg, words, vstart, values}     -> {cfg, words, entries u32[3n]}
/// `cfg` is the device control block (ndx_wah_counts at offset 0); W and D
/// never leave the device until the caller reads them.
struct IndexStages {
  ActorHandle plan, sort, emit, table;
  ActorHandle chain;  // table * emit * sort * plan
};

IndexStages spawn_index_stages(ActorSystem& sys, Device& dev, std::uint32_t row_base = 0);

/// The multi-GPU build's local chain: plan, sort, emit,
/// table and the shard metadata stage, row ids from `row_base`.
/// {keys, wbuf} -> {cfg, wbuf (the words), entries, meta (meta_cap records)}.
struct ShardStages {
  ActorHandle plan, sort, emit, table, meta;
  ActorHandle chain;  // meta * table * emit * sort * plan
};
ShardStages spawn_shard_stages(ActorSystem& sys, Device& dev, std::uint32_t row_base, std::uint32_t meta_cap);

/// Device-resident result of the chain.
struct DeviceIndex {
  std::uint32_t row_count = 0;
  MemRef cfg;      // ndx_wah_counts {words, distinct, min, max} at offset 0
  MemRef words;    // first `words` entries valid
  MemRef entries;  // first 3*`distinct` entries valid
};

/// Runs the chain on device-resident keys; returns without synchronising.
DeviceIndex build_index_device(ActorSystem& sys, const IndexStages& stages, MemRef keys,
                               std::uint32_t row_count);

/// Reads a device index back (waits for its events).
WahIndex fetch_index(const DeviceIndex& d);

/// Builds the per-value bitmap index on the device; identical, word for
/// word, to the reference's reference_index (wah_builder.cpp:38-307).
WahIndex build_index(ActorSystem& sys, Device& dev, std::span<const std::uint32_t> values,
                     unsigned digit_bits = 16);

}  // namespace ndactor::wah
