// Synthetic column generators, bit-identical to the reference's
// (std::mt19937 + uniform_int_distribution, p/tools/ndcli.cpp:144-148;
// the Zipf stream of SURVEY.md Appendix C) because they use the same
// libstdc++ distributions.  The random stream is inherently sequential; the
// Zipf inverse-CDF lookup (the expensive part) runs on all host threads with
// a guide table that returns exactly std::lower_bound's answer.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "ndactor_c.h"

extern "C" {

void ndactor_gen_uniform(uint32_t seed, uint64_t n, uint32_t cardinality, uint32_t* out) {
  std::mt19937 rng(seed);
  std::uniform_int_distribution<uint32_t> pick(0, cardinality ? cardinality - 1 : 0);
  for (uint64_t i = 0; i < n; ++i) out[i] = pick(rng);
}

void ndactor_gen_zipf(uint64_t seed, uint64_t n, uint32_t k, double s, uint32_t* out) {
  if (n == 0 || k == 0) return;
  std::vector<double> cdf(k);
  double acc = 0;
  for (uint32_t i = 0; i < k; ++i) {
    acc += std::pow(double(i + 1), -s);
    cdf[i] = acc;
  }
  for (double& c : cdf) c /= acc;

  // u stream first (sequential), then the lookups in parallel.
  std::vector<double> u(n);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(0.0, 1.0);
  for (uint64_t i = 0; i < n; ++i) u[i] = dist(rng);

  constexpr uint32_t G = 1u << 16;
  std::vector<uint32_t> guide(G + 1);
  for (uint32_t b = 0; b <= G; ++b)
    guide[b] = uint32_t(std::lower_bound(cdf.begin(), cdf.end(), double(b) / G) - cdf.begin());

  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> ts;
  for (unsigned t = 0; t < nt; ++t) {
    ts.emplace_back([&, t] {
      uint64_t lo = n * t / nt, hi = n * (t + 1) / nt;
      for (uint64_t i = lo; i < hi; ++i) {
        double x = u[i];
        uint32_t b = uint32_t(x * G);
        if (b >= G) b = G - 1;
        uint32_t a = guide[b];
        uint32_t e = std::min<uint32_t>(guide[b + 1] + 1, k);
        uint32_t r = uint32_t(std::lower_bound(cdf.begin() + a, cdf.begin() + e, x) - cdf.begin());
        out[i] = std::min<uint32_t>(r, k - 1);
      }
    });
  }
  for (auto& th : ts) th.join();
}

}  // extern "C"

extern "C" {

// The instance stream of the reference's acceptance gate
// (p/tests/acceptance.cpp:56-63): for i in [0, count): rows = 1 + rng() %
// max_rows, then `rows` values from uniform_int(0, cards[i % ncards] - 1),
// all from ONE std::mt19937(seed).  Writes the sizes to `sizes` and the
// concatenated values to `out` (callers size it with sizes from a first
// call with out == nullptr).
void ndactor_gen_instances(uint32_t seed, uint32_t count, const uint32_t* cards,
                           uint32_t ncards, uint32_t max_rows, uint64_t* sizes,
                           uint32_t* out) {
  std::mt19937 rng(seed);
  uint64_t pos = 0;
  for (uint32_t i = 0; i < count; ++i) {
    uint64_t rows = 1 + rng() % max_rows;
    sizes[i] = rows;
    std::uniform_int_distribution<uint32_t> pick(0, cards[i % ncards] - 1);
    for (uint64_t r = 0; r < rows; ++r) {
      uint32_t v = pick(rng);
      if (out) out[pos] = v;
      ++pos;
    }
  }
}

}  // extern "C"
