// The paper's overhead protocols on the B200 device (include/ndactor/bench.hpp).
#include "ndactor/bench.hpp"

#include <cmath>
#include <limits>
#include <numbers>
#include <stdexcept>

#include "ndx.h"

namespace ndactor::bench {

std::vector<float> random_matrix(std::mt19937& rng, std::size_t n) {
  std::uniform_int_distribution<int> digit(0, 9);
  std::vector<float> m(n * n);
  for (float& v : m) v = float(digit(rng));
  return m;
}

KernelDef matmul_kernel() {
  return KernelDef("matmul", [](const LaunchParams& lp) -> int {
    // args: m1, m2 (in), out; the range is n x n
    return ndx_matmul_f32(static_cast<const float*>(lp.ptr[0]), static_cast<const float*>(lp.ptr[1]),
                          static_cast<float*>(lp.ptr[2]), lp.global[0], lp.stream);
  });
}

ActorHandle spawn_matmul(ActorSystem& sys, Device& dev) {
  ComputeActorSpec spec;
  spec.kernel = matmul_kernel();
  spec.args = {ArgSpec::in(ElemType::f32), ArgSpec::in(ElemType::f32), ArgSpec::out(ElemType::f32)};
  spec.range_fn = [](const Message& m) {
    std::size_t n = 1;
    if (!m.empty() && m.at(0).is_array()) n = std::size_t(std::llround(std::sqrt(double(m.at(0).array_length()))));
    return NdRange::grid2(n, n);
  };
  return spawn_compute(sys, dev, std::move(spec));
}

std::vector<float> request_matmul(ActorSystem& sys, const ActorHandle& actor, std::vector<float> m1,
                                  std::vector<float> m2, std::size_t n) {
  Reply r = sys.request(actor, Message::of(std::move(m1), std::move(m2))).await();
  if (is_error(r)) throw std::runtime_error("matmul request failed: " + get_error(r).what);
  std::vector<float> out = std::get<Message>(r).at(0).take_f32s();
  if (out.size() != n * n) throw std::runtime_error("matmul reply has the wrong shape");
  return out;
}

std::vector<float> enqueue_matmul(Device& dev, const std::vector<float>& m1, const std::vector<float>& m2,
                                  std::size_t n) {
  const auto len = std::int64_t(n * n);
  Buffer a = dev.create_buffer_uninit(ElemType::f32, len);
  Buffer b = dev.create_buffer_uninit(ElemType::f32, len);
  Buffer o = dev.create_buffer_uninit(ElemType::f32, len);
  Event wa = dev.enqueue_write(a, m1);
  Event wb = dev.enqueue_write(b, m2);
  Event run = dev.enqueue_kernel(matmul_kernel(), NdRange::grid2(n, n),
                                 {KernelArg::global(a), KernelArg::global(b), KernelArg::global(o)}, {wa, wb});
  std::vector<float> out = dev.read<float>(o, {run});
  dev.free_buffer(a);
  dev.free_buffer(b);
  dev.free_buffer(o);
  return out;
}

double t_quantile_975(std::size_t df) {
  if (df == 0) return std::numeric_limits<double>::infinity();
  const double p = 0.975;
  if (df == 1) return std::tan(std::numbers::pi * (p - 0.5));             // Cauchy
  if (df == 2) return (2 * p - 1) / std::sqrt(2 * p * (1 - p));            // closed form
  // Abramowitz & Stegun 26.7.5: expansion in 1/df around the normal quantile
  const double z = 1.959963984540054, z2 = z * z, v = double(df);
  const double g1 = (z2 + 1) * z / 4;
  const double g2 = ((5 * z2 + 16) * z2 + 3) * z / 96;
  const double g3 = (((3 * z2 + 19) * z2 + 17) * z2 - 15) * z / 384;
  const double g4 = ((((79 * z2 + 776) * z2 + 1482) * z2 - 1920) * z2 - 945) * z / 92160;
  return z + g1 / v + g2 / (v * v) + g3 / (v * v * v) + g4 / (v * v * v * v);
}

LinearFit fit_line(std::span<const double> x, std::span<const double> y) {
  if (x.size() != y.size() || x.size() < 3) throw std::invalid_argument("line fit needs three or more points");
  const double n = double(x.size());
  double sx = 0, sy = 0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    sx += x[i];
    sy += y[i];
  }
  const double mx = sx / n, my = sy / n;
  double sxx = 0, sxy = 0, syy = 0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    const double dx = x[i] - mx, dy = y[i] - my;
    sxx += dx * dx;
    sxy += dx * dy;
    syy += dy * dy;
  }
  if (sxx == 0) throw std::invalid_argument("line fit needs two distinct x values");
  LinearFit f;
  f.slope = sxy / sxx;
  f.intercept = my - f.slope * mx;
  const double ss_res = std::max(0.0, syy - f.slope * sxy);
  f.r2 = syy == 0 ? 1.0 : 1.0 - ss_res / syy;
  const double se = std::sqrt(ss_res / (n - 2) / sxx);
  const double t = t_quantile_975(x.size() - 2);
  f.slope_low = f.slope - t * se;
  f.slope_high = f.slope + t * se;
  return f;
}

}  // namespace ndactor::bench
