// WAH format helpers, restating p/tests/test_wah.cpp:50-256 (CPU only).
#include <cstdio>
#include <random>

#include "harness.hpp"
#include "ndactor/wah.hpp"
#include "ndactor/wah_io.hpp"

using namespace ndactor::wah;

TEST("cpu", "wah format: hand-checked words") {
  CHECK(encode(std::vector<bool>(31, false)) == std::vector<uint32_t>{0x80000001u});
  CHECK(encode(std::vector<bool>(31, true)) == std::vector<uint32_t>{0xc0000001u});
  CHECK(encode(std::vector<bool>(62, false)) == std::vector<uint32_t>{0x80000002u});
  CHECK(encode(std::vector<bool>(93, true)) == std::vector<uint32_t>{0xc0000003u});
  CHECK(encode({true}) == std::vector<uint32_t>{1u});
  CHECK(encode({true, true}) == std::vector<uint32_t>{3u});
  CHECK(encode({}).empty());
  std::vector<bool> b31(32, false);
  b31[31] = true;
  CHECK((encode(b31) == std::vector<uint32_t>{0x80000001u, 1u}));
  CHECK((encode(std::vector<bool>(100, true)) == std::vector<uint32_t>{0xc0000003u, 0x7fu}));
}

TEST("cpu", "wah format: writer merges and splits") {
  CanonicalWriter w;
  w.uniform(false, 1);
  w.chunk(0);
  w.uniform(false, 2);
  CHECK(w.take() == std::vector<uint32_t>{0x80000004u});
  CanonicalWriter ones;
  ones.chunk(kLiteralMask);
  ones.chunk(kLiteralMask);
  CHECK(ones.take() == std::vector<uint32_t>{0xc0000002u});
  CanonicalWriter big;
  big.uniform(false, uint64_t(kLenMask) + 5);
  CHECK((big.take() == std::vector<uint32_t>{0x80000000u | kLenMask, 0x80000005u}));
}

TEST("cpu", "wah format: decode inverts encode; malformed rejected") {
  std::mt19937 rng(7001);
  for (int it = 0; it < 300; ++it) {
    size_t n = 1 + rng() % 400;
    std::bernoulli_distribution bit(std::array<double, 5>{0.0, 0.02, 0.5, 0.98, 1.0}[it % 5]);
    std::vector<bool> bits(n);
    for (size_t i = 0; i < n; ++i) bits[i] = bit(rng);
    CHECK(decode_exact(encode(bits), n) == bits);
  }
  CHECK_THROWS_AS(decode(std::vector<uint32_t>{0x80000000u}), WahError);
  CHECK_THROWS_AS(decode_exact(std::vector<uint32_t>{1u}, 62), WahError);
  CHECK_THROWS_AS(decode_exact(std::vector<uint32_t>{0x80000002u}, 20), WahError);
  CHECK_THROWS_AS(decode_exact(std::vector<uint32_t>{0x40000000u}, 30), WahError);
  CHECK(decode_exact(std::vector<uint32_t>{0x40000000u}, 31)[30]);
}

TEST("cpu", "wah format: rows_for and golden serialized bytes") {
  WahIndex idx;
  idx.row_count = 4;
  idx.entries = {{5, 0, 1}, {7, 1, 1}};
  idx.words = {0x0000000bu, 0x00000004u};
  CHECK((rows_for(idx, 5) == std::vector<uint32_t>{0, 1, 3}));
  CHECK((rows_for(idx, 7) == std::vector<uint32_t>{2}));
  CHECK(rows_for(idx, 6).empty());
  const unsigned char golden[] = {'W', 'A', 'H', '1', 4, 0, 0, 0, 2, 0, 0, 0, 2, 0, 0, 0, 5, 0, 0, 0, 0, 0, 0, 0,
                                  1,   0,   0,   0,   7, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 0x0b, 0, 0, 0, 4, 0, 0, 0};
  auto bytes = serialize_index(idx);
  REQUIRE(bytes.size() == sizeof golden);
  for (size_t i = 0; i < bytes.size(); ++i) CHECK(std::to_integer<unsigned>(bytes[i]) == golden[i]);
  CHECK(parse_index(bytes) == idx);
  bytes.pop_back();
  CHECK_THROWS_AS(parse_index(bytes), WahError);
  WahIndex broken = idx;
  broken.entries[1].length = 9;
  CHECK_THROWS_AS(parse_index(serialize_index(broken)), WahError);
}

TEST("cpu", "wah format: index and value files round-trip") {
  WahIndex idx;
  idx.row_count = 100;
  idx.entries = {{42, 0, 2}};
  idx.words = {0xc0000003u, 0x7fu};
  write_index_file("/tmp/ndactor_t.wah", idx);
  CHECK(read_index_file("/tmp/ndactor_t.wah") == idx);
  std::vector<uint32_t> v{0, 1, 0xffffffffu, 77};
  {
    FILE* f = std::fopen("/tmp/ndactor_t.bin", "wb");
    std::fwrite(v.data(), 4, v.size(), f);
    std::fclose(f);
    f = std::fopen("/tmp/ndactor_t.txt", "w");
    std::fprintf(f, "0\n1\n\n4294967295\n77\n");
    std::fclose(f);
  }
  CHECK(read_values_raw("/tmp/ndactor_t.bin") == v);
  CHECK(read_values_text("/tmp/ndactor_t.txt") == v);
}

// libndactor_verify.so: the reference's CPU ground truth for its own
// consumers (p/tests/test_wah.cpp:132-160 hand vectors)
TEST("cpu", "wah verify library: reference_index hand vectors") {
  const std::vector<uint32_t> a{5, 5, 7, 5};
  WahIndex ia = reference_index(a);
  REQUIRE(ia.entries.size() == 2);
  CHECK(ia.entries[0].value == 5 && ia.entries[0].offset == 0 && ia.entries[0].length == 1);
  CHECK(ia.entries[1].value == 7 && ia.entries[1].offset == 1 && ia.entries[1].length == 1);
  CHECK((ia.words == std::vector<uint32_t>{0xbu, 0x4u}));
  CHECK((reference_index(std::vector<uint32_t>(100, 42)).words == std::vector<uint32_t>{0xc0000003u, 0x7fu}));
  std::vector<uint32_t> c(100, 3);
  c[0] = 9;
  c[99] = 9;
  WahIndex ic = reference_index(c);
  REQUIRE(ic.entries.size() == 2 && ic.entries[1].value == 9);
  const auto b9 = ic.bitmap(ic.entries[1]);
  CHECK((std::vector<uint32_t>(b9.begin(), b9.end()) == std::vector<uint32_t>{0x1u, 0x80000002u, 0x40u}));
  const auto b3 = ic.bitmap(ic.entries[0]);
  CHECK((std::vector<uint32_t>(b3.begin(), b3.end()) == std::vector<uint32_t>{0x7ffffffeu, 0xc0000002u, 0x3fu}));
  CHECK(reference_index(std::vector<uint32_t>{}).entries.empty());
}

TEST("cpu", "wah verify library: reference_index matches rows_for on random columns") {
  std::mt19937 rng(77);
  for (int it = 0; it < 20; ++it) {
    std::uniform_int_distribution<uint32_t> card(1, 200), len(1, 5000);
    const uint32_t k = card(rng);
    std::uniform_int_distribution<uint32_t> pick(0, k - 1);
    std::vector<uint32_t> v(len(rng));
    for (auto& x : v) x = pick(rng) * 7 + 3;
    WahIndex idx = reference_index(v);
    for (const IndexEntry& e : idx.entries) {
      std::vector<uint32_t> want;
      for (uint32_t r = 0; r < v.size(); ++r)
        if (v[r] == e.value) want.push_back(r);
      CHECK(rows_for(idx, e.value) == want);
    }
  }
}
