// ndactor/bench.hpp -- the paper's overhead protocols on the B200 device
// (reference: p/core/include/ndactor/bench.hpp, p/core/src/bench_protocols.cpp;
// acceptance checks 6-7, p/tests/acceptance.cpp:256-330).
#pragma once

#include <cstddef>
#include <random>
#include <span>
#include <vector>

#include "ndactor/compute_actor.hpp"

namespace ndactor::bench {

/// n x n matrix of small integers (digits 0..9) as floats: products and sums
/// stay exact in fp32, so the device result can be compared bit for bit.
std::vector<float> random_matrix(std::mt19937& rng, std::size_t n);

/// The sm_100a matrix product as a kernel definition (ndx_matmul_f32).
KernelDef matmul_kernel();

/// Compute actor answering (m1, m2) -- two value-mode f32 arrays -- with
/// their product; the dimension comes from the first argument's length.
ActorHandle spawn_matmul(ActorSystem& sys, Device& dev);
std::vector<float> request_matmul(ActorSystem& sys, const ActorHandle& actor,
                                  std::vector<float> m1, std::vector<float> m2, std::size_t n);
/// The same product through the raw device API: writes, kernel, read.
std::vector<float> enqueue_matmul(Device& dev, const std::vector<float>& m1,
                                  const std::vector<float>& m2, std::size_t n);

/// Ordinary least squares with a two-sided 95% interval for the slope.
struct LinearFit {
  double slope = 0;
  double intercept = 0;
  double r2 = 0;
  double slope_low = 0;
  double slope_high = 0;
};
LinearFit fit_line(std::span<const double> x, std::span<const double> y);
/// Upper 97.5% quantile of Student's t with df degrees of freedom.
double t_quantile_975(std::size_t df);

}  // namespace ndactor::bench
