// Drop-in check of the C++ wrapper (paper_1607_04091_b200/cpp/gs_b200.hpp):
// the same calls the reference's own tests make (test_freq2wave.cpp,
// test_solver.cpp), run against libgs_b200.so.  Exit 0 on success.
#include <cmath>
#include <cstdio>
#include <random>

#include "gs_b200.hpp"

int main() {
  // jittered 1D db4 operator (test_freq2wave.cpp:144-153 shape)
  gs::SamplingSet pts{1, {}};
  std::mt19937_64 rng(77);
  std::uniform_real_distribution<double> jit(-0.05, 0.05);
  for (int m = 0; m < 64; ++m) pts.coords.push_back(0.225 * (m - 32) + jit(rng));
  gs::Freq2WaveOp op = gs::freq2wave(pts, gs::Family::db4, 4);
  if (op.uniform_fast || op.rows() != 64 || op.cols() != 16) return 1;
  // forward / adjoint pairing (test_freq2wave.cpp:184-194)
  std::uniform_real_distribution<double> u(-1, 1);
  gs::cvec x(16), y(64);
  for (auto& v : x) v = {u(rng), u(rng)};
  for (auto& v : y) v = {u(rng), u(rng)};
  gs::cvec tx = gs::apply_forward(op, x), ty = gs::apply_adjoint(op, y);
  std::complex<double> l = 0, r = 0;
  double nx = 0, ny = 0;
  for (int m = 0; m < 64; ++m) l += tx[m] * std::conj(y[m]), ny += std::norm(y[m]);
  for (int k = 0; k < 16; ++k) r += x[k] * std::conj(ty[k]), nx += std::norm(x[k]);
  if (std::abs(l - r) / std::sqrt(nx * ny) > 1e-12) return 2;
  // in-span recovery (test_solver.cpp:19-33)
  auto [sol, st] = gs::solve_least_squares(op, tx);
  double e = 0;
  for (int k = 0; k < 16; ++k) e += std::norm(sol[k] - x[k]);
  if (!st.converged || std::sqrt(e / nx) > 1e-6 || st.history.size() != (size_t)st.iterations + 1) return 3;
  // error classes (test_freq2wave.cpp:288-294)
  try {
    gs::apply_forward(op, gs::cvec(7));
    return 4;
  } catch (const gs::ShapeError& err) {
    if (err.exit_code() != 4) return 5;
  }
  std::printf("wrapper ok: iterations %d residual %.3e\n", st.iterations, st.residual);
  return 0;
}
