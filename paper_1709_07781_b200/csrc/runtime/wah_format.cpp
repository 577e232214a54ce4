// Host helpers over the WAH word format and the "WAH1" file.
// Behaviour pinned by p/tests/test_wah.cpp (encode/decode known answers,
// canonical writer merging, rows_for truncation, golden serialized bytes)
// and p/core/src/wah_index_io.cpp:30-132 (file layout, value readers).
#include <algorithm>
#include <cstring>
#include <fstream>
#include <iterator>
#include <sstream>

#include "ndactor/wah.hpp"
#include "ndactor/wah_io.hpp"

namespace ndactor::wah {

// ------------------------------------------------------------- writer --

void CanonicalWriter::flush() {
  for (; run_len_ > 0;) {
    const std::uint32_t take = std::uint32_t(std::min<std::uint64_t>(run_len_, kLenMask));
    words_.push_back(make_fill(run_ones_, take));
    run_len_ -= take;
  }
}

void CanonicalWriter::uniform(bool ones, std::uint64_t count) {
  if (!count) return;
  if (run_len_ && run_ones_ != ones) flush();
  run_ones_ = ones;
  run_len_ += count;
}

void CanonicalWriter::chunk(std::uint32_t bits) {
  if (bits == 0 || bits == kLiteralMask) {
    uniform(bits != 0, 1);
    return;
  }
  flush();
  words_.push_back(bits);
}

std::vector<std::uint32_t> CanonicalWriter::take() {
  flush();
  return std::move(words_);
}

// --------------------------------------------------------- codec ------

std::vector<std::uint32_t> encode(const std::vector<bool>& bits) {
  CanonicalWriter w;
  const std::size_t n = bits.size();
  for (std::size_t c = 0; c * kChunkBits < n; ++c) {
    std::uint32_t lit = 0;
    const std::size_t lo = c * kChunkBits, hi = std::min(n, lo + kChunkBits);
    for (std::size_t i = lo; i < hi; ++i) lit |= std::uint32_t(bits[i]) << (i - lo);
    w.chunk(lit);
  }
  return w.take();
}

namespace {
// Calls f(bit_position, value) for every covered bit; returns the coverage.
template <class F>
std::size_t walk_words(std::span<const std::uint32_t> words, F&& f) {
  std::size_t pos = 0;
  for (const std::uint32_t w : words) {
    if (is_fill(w)) {
      if (fill_len(w) == 0) throw WahError("fill word with zero length");
      const std::size_t span = std::size_t(fill_len(w)) * kChunkBits;
      f(pos, span, is_ones_fill(w), 0u, true);
      pos += span;
    } else {
      f(pos, std::size_t(kChunkBits), false, w, false);
      pos += kChunkBits;
    }
  }
  return pos;
}
}  // namespace

std::vector<bool> decode(std::span<const std::uint32_t> words) {
  std::vector<bool> bits;
  walk_words(words, [&](std::size_t, std::size_t span, bool ones, std::uint32_t lit, bool fill) {
    if (fill) {
      bits.insert(bits.end(), span, ones);
    } else {
      for (std::uint32_t i = 0; i < kChunkBits; ++i) bits.push_back((lit >> i) & 1u);
    }
  });
  return bits;
}

std::vector<bool> decode_exact(std::span<const std::uint32_t> words, std::size_t n) {
  std::vector<bool> bits = decode(words);
  if (bits.size() < n) throw WahError("words cover fewer bits than expected");
  if (bits.size() >= n + kChunkBits) throw WahError("words cover a whole chunk beyond the expected bits");
  if (std::find(bits.begin() + std::ptrdiff_t(n), bits.end(), true) != bits.end())
    throw WahError("padding bit is set");
  bits.resize(n);
  return bits;
}

std::vector<std::uint32_t> rows_for(const WahIndex& idx, std::uint32_t value) {
  std::vector<std::uint32_t> rows;
  auto it = std::partition_point(idx.entries.begin(), idx.entries.end(),
                                 [&](const IndexEntry& e) { return e.value < value; });
  if (it == idx.entries.end() || it->value != value) return rows;
  walk_words(idx.bitmap(*it), [&](std::size_t pos, std::size_t span, bool ones, std::uint32_t lit, bool fill) {
    if (fill) {
      if (ones)
        for (std::size_t i = 0; i < span; ++i) rows.push_back(std::uint32_t(pos + i));
    } else {
      for (std::uint32_t b = lit; b; b &= b - 1) rows.push_back(std::uint32_t(pos + __builtin_ctz(b)));
    }
  });
  return rows;
}

bool operator==(const WahIndex& a, const WahIndex& b) {
  if (a.row_count != b.row_count || a.words != b.words || a.entries.size() != b.entries.size())
    return false;
  return std::equal(a.entries.begin(), a.entries.end(), b.entries.begin(),
                    [](const IndexEntry& x, const IndexEntry& y) {
                      return x.value == y.value && x.offset == y.offset && x.length == y.length;
                    });
}

// ----------------------------------------------------------- files -----

namespace {
constexpr char kMagic[4] = {'W', 'A', 'H', '1'};

void put32(std::vector<std::byte>& out, std::uint32_t v) {
  const std::byte b[4] = {std::byte(v), std::byte(v >> 8), std::byte(v >> 16), std::byte(v >> 24)};
  out.insert(out.end(), b, b + 4);
}

struct Reader {
  std::span<const std::byte> in;
  std::size_t pos = 0;
  std::uint32_t u32() {
    if (in.size() - pos < 4) throw WahError("index data is truncated");
    std::uint32_t v = 0;
    for (int i = 3; i >= 0; --i) v = (v << 8) | std::to_integer<std::uint32_t>(in[pos + i]);
    pos += 4;
    return v;
  }
};

std::vector<char> slurp(const std::filesystem::path& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw WahError("cannot open " + path.string());
  return std::vector<char>(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}
}  // namespace

std::vector<std::byte> serialize_index(const WahIndex& idx) {
  std::vector<std::byte> out;
  out.reserve(16 + 12 * idx.entries.size() + 4 * idx.words.size());
  for (char c : kMagic) out.push_back(std::byte(c));
  put32(out, idx.row_count);
  put32(out, std::uint32_t(idx.entries.size()));
  put32(out, std::uint32_t(idx.words.size()));
  for (const IndexEntry& e : idx.entries) {
    put32(out, e.value);
    put32(out, e.offset);
    put32(out, e.length);
  }
  for (std::uint32_t w : idx.words) put32(out, w);
  return out;
}

WahIndex parse_index(std::span<const std::byte> bytes) {
  if (bytes.size() < 4 || std::memcmp(bytes.data(), kMagic, 4) != 0) throw WahError("not a WAH index file");
  Reader r{bytes, 4};
  WahIndex idx;
  idx.row_count = r.u32();
  const std::uint32_t d = r.u32(), w = r.u32();
  idx.entries.resize(d);
  for (IndexEntry& e : idx.entries) {
    e.value = r.u32();
    e.offset = r.u32();
    e.length = r.u32();
    if (std::uint64_t(e.offset) + e.length > w) throw WahError("index entry points past the word array");
  }
  idx.words.resize(w);
  for (std::uint32_t& x : idx.words) x = r.u32();
  if (r.pos != bytes.size()) throw WahError("trailing bytes after index data");
  return idx;
}

void write_index_file(const std::filesystem::path& path, const WahIndex& idx) {
  const std::vector<std::byte> bytes = serialize_index(idx);
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw WahError("cannot open " + path.string() + " for writing");
  f.write(reinterpret_cast<const char*>(bytes.data()), std::streamsize(bytes.size()));
  if (!f) throw WahError("write to " + path.string() + " failed");
}

WahIndex read_index_file(const std::filesystem::path& path) {
  const std::vector<char> raw = slurp(path);
  return parse_index(std::span(reinterpret_cast<const std::byte*>(raw.data()), raw.size()));
}

std::vector<std::uint32_t> read_values_raw(const std::filesystem::path& path) {
  const std::vector<char> raw = slurp(path);
  if (raw.size() % 4) throw WahError(path.string() + " is not a whole number of u32 values");
  std::vector<std::uint32_t> v(raw.size() / 4);
  for (std::size_t i = 0; i < v.size(); ++i) {
    const auto* p = reinterpret_cast<const unsigned char*>(raw.data() + 4 * i);
    v[i] = std::uint32_t(p[0]) | std::uint32_t(p[1]) << 8 | std::uint32_t(p[2]) << 16 |
           std::uint32_t(p[3]) << 24;
  }
  return v;
}

std::vector<std::uint32_t> read_values_text(const std::filesystem::path& path) {
  std::ifstream f(path);
  if (!f) throw WahError("cannot open " + path.string());
  std::vector<std::uint32_t> out;
  std::string line;
  for (std::size_t no = 1; std::getline(f, line); ++no) {
    std::istringstream ls(line);
    std::string tok, extra;
    if (!(ls >> tok)) continue;  // blank line
    const bool digits = !tok.empty() && std::all_of(tok.begin(), tok.end(), ::isdigit);
    if (!digits) throw WahError(path.string() + ":" + std::to_string(no) + ": expected an unsigned integer");
    const unsigned long long v = tok.size() > 10 ? ~0ull : std::stoull(tok);
    if ((ls >> extra) || v > 0xffffffffull)
      throw WahError(path.string() + ":" + std::to_string(no) + ": expected one u32 per line");
    out.push_back(std::uint32_t(v));
  }
  return out;
}

}  // namespace ndactor::wah
