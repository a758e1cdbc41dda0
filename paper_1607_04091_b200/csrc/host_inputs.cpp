// host_inputs.cpp -- input harness for the benchmark configs:
//   * sampling patterns with the reference's exact generators
//     (patterns.cpp:14-74: std::mt19937_64 + std::uniform_real_distribution,
//     so the same libstdc++ yields the same doubles);
//   * exact Voronoi density-compensation weights in O(M log M): the cell of
//     point m is clipped (the same half-plane clip as weights.cpp:20-38) only
//     against neighbours in expanding bucket rings, stopping once every
//     unprocessed point is farther than twice the cell's farthest vertex --
//     beyond that no bisector can cut the cell, so the polygon equals the
//     reference's clip against all M points (weights.cpp:59-70).
//   * the density report, the bench harness's seeded coefficients and the
//     truncated-cosine test signal (weights.cpp:135-176, bench.cpp:30-36,
//     signals.cpp:12-37) for the command-line front end.
// Multi-threaded with std::thread.  Not on the timed path.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "voronoi_common.h"

namespace {

struct P2 {
  double x, y;
};

void clip(std::vector<P2>& poly, std::vector<P2>& tmp, P2 mid, P2 a) {  // weights.cpp:20-38
  tmp.clear();
  size_t n = poly.size();
  for (size_t i = 0; i < n; ++i) {
    const P2& cur = poly[i];
    const P2& nxt = poly[(i + 1) % n];
    double dc = a.x * (cur.x - mid.x) + a.y * (cur.y - mid.y);
    double dn = a.x * (nxt.x - mid.x) + a.y * (nxt.y - mid.y);
    if (dc <= 0) tmp.push_back(cur);
    if ((dc < 0 && dn > 0) || (dc > 0 && dn < 0)) {
      double t = dc / (dc - dn);
      tmp.push_back({cur.x + t * (nxt.x - cur.x), cur.y + t * (nxt.y - cur.y)});
    }
  }
  poly.swap(tmp);
}

double area(const std::vector<P2>& poly) {  // weights.cpp:40-49
  double acc = 0.0;
  size_t n = poly.size();
  for (size_t i = 0; i < n; ++i) acc += poly[i].x * poly[(i + 1) % n].y - poly[(i + 1) % n].x * poly[i].y;
  return 0.5 * std::abs(acc);
}

thread_local std::string g_in_err;

}  // namespace

extern "C" {

const char* gs_inputs_last_error(void) { return g_in_err.c_str(); }

// patterns.cpp:25-44
int gs_gen_grid(int64_t M, double eps, int dim, double* out) {
  if (M < 1 || !(eps > 0) || (dim != 1 && dim != 2)) {
    g_in_err = "bad grid parameters";
    return 5;
  }
  std::vector<double> axis(M);
  double half = (double)M / 2.0;
  for (int64_t m = 0; m < M; ++m) axis[m] = eps * ((double)m - half);
  if (dim == 1) {
    std::memcpy(out, axis.data(), M * sizeof(double));
    return 0;
  }
  int64_t k = 0;
  for (double x : axis)
    for (double y : axis) {
      out[k++] = x;
      out[k++] = y;
    }
  return 0;
}

// patterns.cpp:46-56
int gs_gen_jitter(int64_t M, double eps, double eta, uint64_t seed, int dim, double* out) {
  if (!(eta >= 0) || eta >= eps / 2) {
    g_in_err = "eta must satisfy 0 <= eta < epsilon/2";
    return 5;
  }
  int rc = gs_gen_grid(M, eps, dim, out);
  if (rc) return rc;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> shift(-eta, eta);
  int64_t n = M * (dim == 2 ? M * 2 : 1);
  for (int64_t i = 0; i < n; ++i) out[i] += shift(rng);
  if (dim == 1) std::sort(out, out + M);
  return 0;
}

// patterns.cpp:58-74
int gs_gen_spiral(int turns, double ppt, double K, double* out) {
  if (turns < 1 || !(ppt > 0) || !(K > 0)) {
    g_in_err = "bad spiral parameters";
    return 5;
  }
  long long count = std::llround(turns * ppt);
  for (long long i = 0; i < count; ++i) {
    double t = (double)i / ppt;
    double radius = K * t / (double)turns;
    double angle = 2.0 * 3.14159265358979323846 * t;
    out[2 * i] = radius * std::cos(angle);
    out[2 * i + 1] = radius * std::sin(angle);
  }
  return 0;
}

// Voronoi cells clipped to [-K, K]^dim (weights.cpp:95-133), exact, fast.
// mu[m] = cell measure; rad[m] (optional) = farthest cell vertex from point m,
// i.e. the largest distance from a vertex of cell m to its nearest sample
// (weights.cpp:135-171 takes the supremum of these over all cells).
// bucket grid of the 2D cells (~2 points per bucket) + the reference's input
// checks (weights.cpp:73-90: range, duplicates); shared with gs_voronoi.cu
extern "C++" int vor_grid_build(int64_t M, const double* coords, double K, std::vector<int64_t>& start,
                                std::vector<int64_t>& idx, int& G, double& h) {
  for (int64_t m = 0; m < M; ++m)
    if (std::abs(coords[2 * m]) > K || std::abs(coords[2 * m + 1]) > K) {
      g_in_err = "point outside the bandwidth region";
      return 5;
    }
  // bucket grid, ~2 points per bucket on average
  G = std::max(1, (int)std::sqrt((double)M / 2.0));
  h = 2.0 * K / G;
  auto cell = [&](double v) { return std::min(G - 1, std::max(0, (int)std::floor((v + K) / h))); };
  start.assign((size_t)G * G + 1, 0);
  idx.assign(M, 0);
  for (int64_t m = 0; m < M; ++m) start[(size_t)cell(coords[2 * m + 1]) * G + cell(coords[2 * m]) + 1]++;
  for (size_t i = 1; i < start.size(); ++i) start[i] += start[i - 1];
  {
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (int64_t m = 0; m < M; ++m) idx[fill[(size_t)cell(coords[2 * m + 1]) * G + cell(coords[2 * m])]++] = m;
  }
  // duplicates (same bucket) -> reference DomainError
  for (size_t b = 0; b + 1 < start.size(); ++b)
    for (int64_t i = start[b]; i < start[b + 1]; ++i)
      for (int64_t j = i + 1; j < start[b + 1]; ++j)
        if (coords[2 * idx[i]] == coords[2 * idx[j]] && coords[2 * idx[i] + 1] == coords[2 * idx[j] + 1]) {
          g_in_err = "degenerate input: duplicate sample points";
          return 5;
        }
  return 0;
}

static int voronoi_cells(int dim, int64_t M, const double* coords, double K, double* mu, double* rad, int nthreads) {
  if (!(K > 0)) {
    g_in_err = "K must be positive";
    return 5;
  }
  if (M <= 0) {
    g_in_err = "empty point set";
    return 4;
  }
  if (dim == 1) {
    std::vector<int64_t> order(M);
    for (int64_t i = 0; i < M; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return coords[a] < coords[b]; });
    for (int64_t i = 1; i < M; ++i)
      if (coords[order[i]] == coords[order[i - 1]]) {
        g_in_err = "degenerate input: duplicate sample points";
        return 5;
      }
    if (coords[order[0]] < -K || coords[order[M - 1]] > K) {
      g_in_err = "point outside the bandwidth region";
      return 5;
    }
    for (int64_t i = 0; i < M; ++i) {
      double lo = i == 0 ? -K : 0.5 * (coords[order[i - 1]] + coords[order[i]]);
      double hi = i + 1 == M ? K : 0.5 * (coords[order[i]] + coords[order[i + 1]]);
      if (mu) mu[order[i]] = hi - lo;
      // density candidates (weights.cpp:147-150): the region ends, half gaps
      if (rad) rad[order[i]] = std::max(i == 0 ? coords[order[0]] + K : 0.0,
                                        i + 1 == M ? K - coords[order[i]]
                                                   : 0.5 * (coords[order[i + 1]] - coords[order[i]]));
    }
    return 0;
  }
  std::vector<int64_t> start, idx;
  int G = 1;
  double h = 0.0;
  {
    const int rc = vor_grid_build(M, coords, K, start, idx, G, h);
    if (rc) return rc;
  }
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  std::atomic<int64_t> next(0);
  const VorGrid grid{coords, start.data(), idx.data(), M, G, K, h};
  auto worker = [&]() {
    // per-cell routine shared with the GPU kernel (voronoi_common.h); buffers grow on overflow
    int capv = 256, capc = 1024;
    std::vector<double> px(capv), py(capv), qx(capv), qy(capv), cd(capc);
    std::vector<int64_t> cj(capc);
    const int64_t chunk = 256;
    for (;;) {
      int64_t lo = next.fetch_add(chunk);
      if (lo >= M) break;
      int64_t hi = std::min(M, lo + chunk);
      for (int64_t m = lo; m < hi; ++m) {
        double mu_m = 0.0, rad_m = 0.0;
        while (vor_cell(grid, m, px.data(), py.data(), qx.data(), qy.data(), capv, cd.data(), cj.data(), capc,
                        &mu_m, &rad_m) != VOR_OK) {
          capv *= 2;
          capc *= 2;
          px.resize(capv);
          py.resize(capv);
          qx.resize(capv);
          qy.resize(capv);
          cd.resize(capc);
          cj.resize(capc);
        }
        if (mu) mu[m] = mu_m;
        if (rad) rad[m] = rad_m;
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) th.emplace_back(worker);
  for (auto& t : th) t.join();
  return 0;
}

int gs_voronoi_weights(int dim, int64_t M, const double* coords, double K, double* mu, int nthreads) {
  return voronoi_cells(dim, M, coords, K, mu, nullptr, nthreads);
}

// density(samples, K) (weights.cpp:135-176): delta_raw = sup over Y_K of the
// distance to the nearest sample, attained at a vertex of the clipped
// tessellation -- the farthest vertex of some cell from that cell's own point.
int gs_density(int dim, int64_t M, const double* coords, double K, double* delta_raw, int nthreads) {
  std::vector<double> rad(M > 0 ? M : 1);
  const int rc = voronoi_cells(dim, M, coords, K, nullptr, rad.data(), nthreads);
  if (rc) return rc;
  double d = 0.0;
  for (int64_t m = 0; m < M; ++m) d = std::max(d, rad[m]);
  *delta_raw = d;
  return 0;
}

// bench.cpp:30-36: x_k = (U(-1,1), U(-1,1)) from mt19937_64(seed ^ golden ratio)
int gs_seeded_coefficients(int64_t n, uint64_t seed, double* out) {
  if (n < 0) {
    g_in_err = "negative count";
    return 4;
  }
  std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ull);
  std::uniform_real_distribution<double> unit(-1.0, 1.0);
  for (int64_t k = 0; k < n; ++k) {
    const double re = unit(rng);
    const double im = unit(rng);
    out[2 * k] = re;
    out[2 * k + 1] = im;
  }
  return 0;
}

// signals.cpp:12-37: analytic transform of cos(2 pi x) on [-1/2, 0)
int gs_truncated_cosine(int64_t M, const double* xi, double* out) {
  const double pi = 3.14159265358979323846;
  auto g = [&](double a, double& re, double& im) {  // (e^{i pi a} - 1) / (2 pi i a), 1/2 at a = 0
    if (a == 0.0) {
      re = 0.5;
      im = 0.0;
      return;
    }
    const double nr = std::cos(pi * a) - 1.0, ni = std::sin(pi * a);
    const double d = 2.0 * pi * a;  // (nr + i ni) / (i d) = ni / d - i nr / d
    re = ni / d;
    im = -nr / d;
  };
  for (int64_t m = 0; m < M; ++m) {
    double ar, ai, br, bi;
    g(xi[m] - 1.0, ar, ai);
    g(xi[m] + 1.0, br, bi);
    out[2 * m] = 0.5 * (ar + br);
    out[2 * m + 1] = 0.5 * (ai + bi);
  }
  return 0;
}

}  // extern "C"
