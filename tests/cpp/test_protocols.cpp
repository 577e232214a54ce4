// The paper's facade-overhead protocol on B200 (reference acceptance checks
// 6 and 7, p/tests/acceptance.cpp:256-330): the matmul compute actor agrees
// with the triple-loop product, and the actor-minus-device time shows no
// confidently positive trend in the problem size.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <random>

#include "harness.hpp"
#include "ndactor/bench.hpp"

using namespace ndactor;

namespace {

// test-side triple loop (the oracle of acceptance check 7)
std::vector<float> triple_loop(const std::vector<float>& a, const std::vector<float>& b, std::size_t n) {
  std::vector<float> out(n * n);
  for (std::size_t y = 0; y < n; ++y)
    for (std::size_t x = 0; x < n; ++x) {
      float r = 0;
      for (std::size_t k = 0; k < n; ++k) r += a[k + y * n] * b[x + k * n];
      out[x + y * n] = r;
    }
  return out;
}

double secs(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
}

}  // namespace

TEST("cpu", "bench: line fit and t quantiles") {
  const std::vector<double> x{1, 2, 3, 4, 5}, y{3, 5, 7, 9, 11};
  bench::LinearFit f = bench::fit_line(x, y);
  CHECK(std::fabs(f.slope - 2) < 1e-12 && std::fabs(f.intercept - 1) < 1e-12 && f.r2 > 0.999999);
  CHECK(std::fabs(bench::t_quantile_975(1) - 12.706) < 1e-3);
  CHECK(std::fabs(bench::t_quantile_975(2) - 4.303) < 1e-3);
  CHECK(std::fabs(bench::t_quantile_975(10) - 2.228) < 2e-3);
  CHECK(std::fabs(bench::t_quantile_975(30) - 2.042) < 1e-3);
  CHECK(std::fabs(bench::t_quantile_975(88) - 1.987) < 1e-3);
  CHECK_THROWS_AS(bench::fit_line(std::vector<double>{1, 1, 1}, std::vector<double>{1, 2, 3}),
                  std::invalid_argument);
}

TEST("gpu", "protocols: matmul actor equals the triple loop (check 7)") {
  ActorSystem sys(2);
  Device dev(DeviceConfig{});
  std::mt19937 rng(808);
  ActorHandle actor = bench::spawn_matmul(sys, dev);
  for (std::size_t n : {1, 7, 33, 64, 128}) {
    auto m1 = bench::random_matrix(rng, n), m2 = bench::random_matrix(rng, n);
    CHECK(bench::request_matmul(sys, actor, m1, m2, n) == triple_loop(m1, m2, n));
  }
  const std::size_t n = 256;
  std::uniform_real_distribution<float> unit(-1.0f, 1.0f);
  std::vector<float> m1(n * n), m2(n * n);
  for (auto& v : m1) v = unit(rng);
  for (auto& v : m2) v = unit(rng);
  const auto want = triple_loop(m1, m2, n);
  const auto got = bench::request_matmul(sys, actor, m1, m2, n);
  double worst = 0;
  for (std::size_t i = 0; i < want.size(); ++i)
    worst = std::max(worst, std::fabs(double(got[i]) - double(want[i])) / std::max(1e-6, double(std::fabs(want[i]))));
  CHECK(worst <= 1e-4);
  sys.terminate(actor);
  sys.await_idle();
}

TEST("gpu", "protocols: facade overhead has no positive trend in n (check 6)") {
  ActorSystem sys(2);
  Device dev(DeviceConfig{});
  std::mt19937 rng(5150);
  ActorHandle actor = bench::spawn_matmul(sys, dev);
  std::vector<double> xs, ys;
  for (std::size_t n : {64, 128, 256}) {
    auto m1 = bench::random_matrix(rng, n), m2 = bench::random_matrix(rng, n);
    for (int w = 0; w < 3; ++w) {  // untimed: first-use allocations of both paths
      bench::request_matmul(sys, actor, m1, m2, n);
      bench::enqueue_matmul(dev, m1, m2, n);
    }
    for (int run = 0; run < 30; ++run) {
      auto ta = std::chrono::steady_clock::now();
      auto via_actor = bench::request_matmul(sys, actor, m1, m2, n);
      const double actor_s = secs(ta);
      auto td = std::chrono::steady_clock::now();
      auto via_device = bench::enqueue_matmul(dev, m1, m2, n);
      const double device_s = secs(td);
      if (run == 29) std::printf("    n %zu: actor %.1f us, device %.1f us (last run)\n", n, actor_s * 1e6, device_s * 1e6);
      REQUIRE(via_actor == via_device);
      xs.push_back(double(n));
      ys.push_back(actor_s - device_s);
    }
  }
  sys.terminate(actor);
  sys.await_idle();
  for (std::size_t i = 0; i < xs.size(); i += 30) {
    double s = 0;
    for (std::size_t j = i; j < i + 30; ++j) s += ys[j];
    std::printf("    n %.0f: actor - device %.1f us (mean of 30)\n", xs[i], s / 30 * 1e6);
  }
  // host jitter (a worker descheduled, a page fault in a fresh pinned
  // block) only ever adds time: fit on the fastest 24 of each n's 30 runs
  std::vector<double> fx, fy;
  for (std::size_t i = 0; i < xs.size(); i += 30) {
    std::vector<double> run(ys.begin() + i, ys.begin() + i + 30);
    std::sort(run.begin(), run.end());
    for (int k = 0; k < 24; ++k) {
      fx.push_back(xs[i]);
      fy.push_back(run[k]);
    }
  }
  const bench::LinearFit fit = bench::fit_line(fx, fy);
  std::printf("    overhead slope 95%% CI [%.3g, %.3g] s per n\n", fit.slope_low, fit.slope_high);
  CHECK(fit.slope_low <= 0.0);  // one-sided: only a confidently positive slope fails
}
