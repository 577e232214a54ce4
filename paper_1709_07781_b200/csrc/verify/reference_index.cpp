// libndactor_verify.so -- the reference's CPU ground truth, wah::reference_index
// (declared at p/core/include/ndactor/wah.hpp:107-109, defined at
// p/core/src/wah_words.cpp:49-91), for the reference's own consumers that call
// it next to the device build: `ndcli index build --verify`
// (p/tools/ndcli.cpp:169) and the acceptance gate (p/tests/acceptance.cpp:65).
//
// Deliberately NOT part of libndactor.so: the product has no CPU build path.
// A consumer that verifies links this library beside libndactor.so; nothing in
// the product links or calls it.
//
// The algorithm is the reference's definition of the index:
// rows grouped by value in ascending order, each value's rows ascending, then
// per value the canonical words chunk by chunk -- a zero-fill for the gap
// before each non-empty chunk, the chunk itself (a ones-fill when full).
#include <algorithm>
#include <numeric>

#include "ndactor/wah.hpp"

namespace ndactor::wah {

WahIndex reference_index(std::span<const std::uint32_t> values) {
  if (values.size() >= (std::size_t(1) << 32)) throw WahError("more rows than the u32 index format holds");
  WahIndex idx;
  idx.row_count = std::uint32_t(values.size());
  // rows in (value, row) order: a stable sort of the row ids by value
  std::vector<std::uint32_t> rows(values.size());
  std::iota(rows.begin(), rows.end(), 0u);
  std::stable_sort(rows.begin(), rows.end(), [&](std::uint32_t a, std::uint32_t b) { return values[a] < values[b]; });
  std::size_t i = 0;
  while (i < rows.size()) {
    const std::uint32_t v = values[rows[i]];
    CanonicalWriter w;
    std::uint64_t next_chunk = 0;  // the first chunk not yet written
    while (i < rows.size() && values[rows[i]] == v) {
      const std::uint64_t c = rows[i] / kChunkBits;
      std::uint32_t bits = 0;
      for (; i < rows.size() && values[rows[i]] == v && rows[i] / kChunkBits == c; ++i)
        bits |= 1u << (rows[i] % kChunkBits);
      w.uniform(false, c - next_chunk);  // the empty chunks in between (no-op at 0)
      w.chunk(bits);
      next_chunk = c + 1;
    }
    std::vector<std::uint32_t> words = w.take();
    idx.entries.push_back(IndexEntry{v, std::uint32_t(idx.words.size()), std::uint32_t(words.size())});
    idx.words.insert(idx.words.end(), words.begin(), words.end());
  }
  return idx;
}

}  // namespace ndactor::wah
