// ndactor/wah_shard.hpp -- multi-GPU build: row shards and the boundary merge
// (SURVEY.md section 8(e), Appendix B).
//
// Shard g holds rows [S_g, S_{g+1}) with S_g a multiple of 31 and is built
// with global row ids (row_base = S_g), so its local index differs from its
// slice of the global index only at the ends of each value's piece.  The plan
// below works on per-value metadata only (a few MB at 8 x 65,536 values); the
// words themselves are moved by ndx_wah_assemble on the GPU.
#pragma once

#include <cstdint>
#include <span>
#include <utility>
#include <vector>

#include "ndactor/wah.hpp"
#include "ndx.h"

namespace ndactor::wah {

/// S_0 = 0 < S_1 < ... < S_G = n, every inner bound a multiple of 31, chunk
/// counts as even as possible.
std::vector<std::uint64_t> shard_bounds(std::uint64_t n, std::uint32_t shards);

struct MergePlan {
  std::vector<IndexEntry> entries;            // union of values, ascending
  std::vector<std::vector<ndx_piece>> pieces;  // [shard][local entry]
  std::uint64_t words = 0;                    // total merged words
};

/// Appendix B: per value, in shard order, the first piece keeps a leading
/// zero-fill of f chunks; a later piece gets a zero-fill of the gap to the
/// previous piece, or -- at gap 0 when both sides are ones-fills -- one fused
/// ones-fill that replaces the previous last word and its own first word.
MergePlan plan_merge(std::span<const std::span<const ndx_shard_meta>> shards);

/// The same, writing straight into caller storage: entries_out (capacity:
/// the total record count) and pieces_out[g][i] for record i of shard g.
/// Returns the merged (entries, words) counts.
std::pair<std::uint64_t, std::uint64_t> plan_merge_into(
    std::span<const std::span<const ndx_shard_meta>> shards, IndexEntry* entries_out,
    std::span<ndx_piece* const> pieces_out);

}  // namespace ndactor::wah
