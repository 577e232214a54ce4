// Row shards and the shard boundary merge plan (include/ndactor/wah_shard.hpp).
#include "ndactor/wah_shard.hpp"

#include <algorithm>
#include <string>

namespace ndactor::wah {

std::vector<std::uint64_t> shard_bounds(std::uint64_t n, std::uint32_t shards) {
  if (shards == 0) throw WahError("shard_bounds: zero shards");
  const std::uint64_t chunks = (n + kChunkBits - 1) / kChunkBits;
  std::vector<std::uint64_t> b(shards + 1);
  for (std::uint32_t g = 0; g <= shards; ++g) {
    const std::uint64_t c = chunks * g / shards;
    b[g] = std::min<std::uint64_t>(c * kChunkBits, n);
  }
  b[shards] = n;
  return b;
}

namespace {

// Where the value's current last word lives, so a fused ones-fill can
// replace it.
struct LastWord {
  ndx_piece* piece = nullptr;
  bool is_lead = false;
  std::uint32_t ones = 0;  // its ones-fill length, 0 if it is not a ones-fill
};

}  // namespace

std::pair<std::uint64_t, std::uint64_t> plan_merge_into(
    std::span<const std::span<const ndx_shard_meta>> shards, IndexEntry* entries_out,
    std::span<ndx_piece* const> pieces_out) {
  const std::size_t G = shards.size();
  if (pieces_out.size() != G) throw WahError("plan_merge: one piece array per shard");
  for (std::size_t g = 0; g < G; ++g)
    for (std::size_t i = 1; i < shards[g].size(); ++i)
      if (shards[g][i].value <= shards[g][i - 1].value)
        throw WahError("plan_merge: shard " + std::to_string(g) + " values not ascending");
  std::vector<std::size_t> head(G, 0);
  std::uint64_t out = 0, ne = 0;
  for (;;) {
    // next value: the smallest head over the shards (G is small)
    bool any = false;
    std::uint32_t v = 0;
    for (std::size_t g = 0; g < G; ++g)
      if (head[g] < shards[g].size() && (!any || shards[g][head[g]].value < v)) {
        v = shards[g][head[g]].value;
        any = true;
      }
    if (!any) break;
    std::uint64_t len = 0;
    LastWord last;
    std::uint32_t prev_l = 0;
    bool first = true;
    for (std::size_t g = 0; g < G; ++g) {
      if (head[g] >= shards[g].size() || shards[g][head[g]].value != v) continue;
      const ndx_shard_meta& m = shards[g][head[g]];
      ndx_piece& p = pieces_out[g][head[g]];
      ++head[g];
      if (m.body_len == 0) throw WahError("plan_merge: empty body");
      p = ndx_piece{0, m.body_off, m.body_len, 0, 0};
      if (first) {
        if (m.f > 0) p.lead = make_fill(false, m.f);
      } else {
        if (m.f <= prev_l) throw WahError("plan_merge: shards overlap in chunks");
        const std::uint32_t gap = m.f - prev_l - 1;
        if (gap > 0) {
          p.lead = make_fill(false, gap);
        } else if (last.ones > 0 && m.a > 0) {
          // fuse: drop the previous last word and this body's first word
          if (last.is_lead)
            last.piece->lead = 0;
          else
            last.piece->src_len -= 1;
          --len;
          p.lead = make_fill(true, last.ones + m.a);
          p.src_off += 1;
          p.src_len -= 1;
        }
      }
      first = false;
      p.dst = out + len;  // absolute: the value's offset is `out`
      len += (p.lead ? 1u : 0u) + p.src_len;
      if (p.src_len > 0)
        last = LastWord{&p, false, m.z};
      else
        last = LastWord{&p, true, is_ones_fill(p.lead) ? fill_len(p.lead) : 0u};
      prev_l = m.l;
    }
    if (out + len > 0xffffffffull) throw WahError("plan_merge: index exceeds u32 word offsets");
    entries_out[ne++] = IndexEntry{v, std::uint32_t(out), std::uint32_t(len)};
    out += len;
  }
  return {ne, out};
}

MergePlan plan_merge(std::span<const std::span<const ndx_shard_meta>> shards) {
  MergePlan plan;
  std::size_t total = 0;
  plan.pieces.resize(shards.size());
  std::vector<ndx_piece*> outs(shards.size());
  for (std::size_t g = 0; g < shards.size(); ++g) {
    plan.pieces[g].resize(shards[g].size());
    outs[g] = plan.pieces[g].data();
    total += shards[g].size();
  }
  plan.entries.resize(total);
  auto [ne, nw] = plan_merge_into(shards, plan.entries.data(), outs);
  plan.entries.resize(ne);
  plan.words = nw;
  return plan;
}

}  // namespace ndactor::wah
