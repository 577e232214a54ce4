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

MergePlan plan_merge(std::span<const std::span<const ndx_shard_meta>> shards) {
  const std::size_t G = shards.size();
  MergePlan plan;
  plan.pieces.resize(G);
  std::size_t total = 0;
  for (std::size_t g = 0; g < G; ++g) {
    plan.pieces[g].resize(shards[g].size());
    total += shards[g].size();
    for (std::size_t i = 1; i < shards[g].size(); ++i)
      if (shards[g][i].value <= shards[g][i - 1].value)
        throw WahError("plan_merge: shard " + std::to_string(g) + " values not ascending");
  }
  plan.entries.reserve(total);
  std::vector<std::size_t> head(G, 0);
  std::vector<std::pair<std::size_t, std::size_t>> group;
  std::vector<std::pair<ndx_piece*, std::uint64_t>> placed;
  std::uint64_t out = 0;
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
    group.clear();
    for (std::size_t g = 0; g < G; ++g)
      if (head[g] < shards[g].size() && shards[g][head[g]].value == v) group.emplace_back(g, head[g]++);

    std::uint64_t len = 0;
    LastWord last;
    std::uint32_t prev_l = 0;
    placed.clear();
    for (std::size_t k = 0; k < group.size(); ++k) {
      const ndx_shard_meta& m = shards[group[k].first][group[k].second];
      ndx_piece& p = plan.pieces[group[k].first][group[k].second];
      p = ndx_piece{0, m.body_off, m.body_len, 0, 0};
      if (m.body_len == 0) throw WahError("plan_merge: empty body");
      if (k == 0) {
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
      placed.emplace_back(&p, len);
      len += (p.lead ? 1u : 0u) + p.src_len;
      if (p.src_len > 0)
        last = LastWord{&p, false, m.z};
      else
        last = LastWord{&p, true, is_ones_fill(p.lead) ? fill_len(p.lead) : 0u};
      prev_l = m.l;
    }
    for (auto& [p, r] : placed) p->dst = out + r;
    if (out + len > 0xffffffffull) throw WahError("plan_merge: index exceeds u32 word offsets");
    plan.entries.push_back(IndexEntry{v, std::uint32_t(out), std::uint32_t(len)});
    out += len;
  }
  plan.words = out;
  return plan;
}

}  // namespace ndactor::wah
