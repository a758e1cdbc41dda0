// host_math.h -- host-side restatements of the reference's small helpers the
// routes share (freq2wave.cpp:15-37, nufft.cpp:163-171, 389-400).
#pragma once
#include <cmath>
#include <algorithm>
#include <cstddef>

#include "gs_common.cuh"
#include "host_common.cuh"

namespace gsb {

inline double wrap_half_open(double z) {  // freq2wave.cpp:15-19
  double w = z - std::floor(z + 0.5);
  if (w >= 0.5) w -= 1.0;
  return w;
}

inline bool detect_uniform(const double* zeta, size_t M, long long n, double* eps_out) {  // freq2wave.cpp:22-37
  if (M < 2 || (long long)M < n) return false;
  double spacing = zeta[1] - zeta[0];
  if (spacing <= 0.0) return false;
  double eps = spacing * (double)n;
  double inv = 1.0 / eps;
  if (std::abs(inv - std::round(inv)) > 1e-9 || std::round(inv) < 1.0) return false;
  double half_m = (double)M / 2.0;
  for (size_t m = 0; m < M; ++m) {
    double expect = eps / (double)n * ((double)m - half_m);
    if (std::abs(zeta[m] - expect) > 1e-12) return false;
  }
  *eps_out = eps;
  return true;
}

inline double kb_transform(double nu, int w, double beta) {  // nufft.cpp:163-171
  double t = beta * beta - (GS_TWO_PI * w * nu) * (GS_TWO_PI * w * nu);
  if (t > 0) {
    double s = std::sqrt(t);
    return 2.0 * w * std::sinh(s) / s;
  }
  double s = std::sqrt(-t);
  return 2.0 * w * std::sin(s) / s;
}

struct UniSetup {
  long long inv_eps, q, n2;
};
inline UniSetup uniform_setup(long long M, double eps, long long N) {  // nufft.cpp:389-400
  if (eps <= 0.0) fail(GS_ERR_DOMAIN, "epsilon must be positive");
  double inv = 1.0 / eps;
  long long inv_eps = std::llround(inv);
  if (inv_eps < 1 || std::abs(inv - (double)inv_eps) > 1e-9) fail(GS_ERR_DOMAIN, "1/epsilon must be a positive integer");
  if (M < N) fail(GS_ERR_DOMAIN, "uniform reduction requires M >= N");
  long long per = N * inv_eps;
  long long q = (M + per - 1) / per;
  return {inv_eps, q, q * per};
}


// beta of the Kaiser-Bessel window (nufft.cpp:201-206)
inline double kb_beta(double sigma, int w) {
  const double width = 2.0 * w;
  const double t = (width / sigma) * (width / sigma) * (sigma - 0.5) * (sigma - 0.5) - 0.8;
  return GS_PI * std::sqrt(std::max(t, 1.0));
}

}  // namespace gsb
