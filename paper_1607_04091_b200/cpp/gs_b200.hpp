// gs_b200.hpp -- header-only C++ drop-in for the reference operator API
// (namespace gs, /root/reference/proj/include/gs/{nufft,freq2wave,solver,error}.hpp)
// over the C-ABI of include/gs_b200.h.  A caller of gs::freq2wave /
// gs::apply_forward / gs::apply_adjoint / gs::solve_least_squares recompiles
// against this header and links libgs_b200.so; vectors stay
// std::vector<std::complex<double>> (host), errors stay gs::Error subclasses
// with the reference's exit codes (error.hpp:9-41).
//
// Differences from the reference, all additive: Freq2WaveOp is a move-only
// handle to device-resident state (the reference's is move-only too because of
// NfftPlan, nufft.hpp:41-62); the factor fields are read through
// op.factors(axis) instead of public Eigen members.
#pragma once

#include <cmath>
#include <complex>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/gs_b200.h"

namespace gs {

using cd = std::complex<double>;
using cvec = std::vector<cd>;

enum class ErrorClass { usage = 2, file_format = 3, shape = 4, domain = 5, numerical = 6 };

class Error : public std::runtime_error {
 public:
  Error(ErrorClass cls, const std::string& msg) : std::runtime_error(msg), cls_(cls) {}
  ErrorClass error_class() const { return cls_; }
  int exit_code() const { return static_cast<int>(cls_); }

 private:
  ErrorClass cls_;
};
struct UsageError : Error {
  explicit UsageError(const std::string& m) : Error(ErrorClass::usage, m) {}
};
struct ShapeError : Error {
  explicit ShapeError(const std::string& m) : Error(ErrorClass::shape, m) {}
};
struct DomainError : Error {
  explicit DomainError(const std::string& m) : Error(ErrorClass::domain, m) {}
};
struct NumericalError : Error {
  explicit NumericalError(const std::string& m) : Error(ErrorClass::numerical, m) {}
};
// CUDA runtime failures have no reference class; they surface as numerical (6)
struct DeviceError : Error {
  explicit DeviceError(const std::string& m) : Error(ErrorClass::numerical, m) {}
};

inline void check(int rc) {
  if (rc == GS_OK) return;
  const std::string m = gs_last_error();
  switch (rc) {
    case GS_ERR_USAGE: throw UsageError(m);
    case GS_ERR_SHAPE: throw ShapeError(m);
    case GS_ERR_DOMAIN: throw DomainError(m);
    case GS_ERR_NUMERICAL: throw NumericalError(m);
    default: throw DeviceError(m);
  }
}

enum class Family { haar, db2, db3, db4, db5, db6, db7, db8 };  // scaling.hpp:10
inline int family_p(Family f) { return f == Family::haar ? 1 : static_cast<int>(f) + 1; }

struct SamplingSet {  // nufft.hpp:16-23
  int dim = 1;
  std::vector<double> coords;
  size_t size() const { return coords.size() / static_cast<size_t>(dim); }
};

struct Freq2WaveOptions {  // freq2wave.hpp:12-24
  std::optional<double> bandwidth;
  std::vector<double> weights;
  double sigma = 2.0;
  int w = 6;
  int boundary_depth = 30;
  int product_terms = 48;
  bool allow_uniform_fast_path = true;
  bool allow_tensor_route = false;  // B200 addition (opt-in): exact route for uniform 2D grids
  int device = 0;
};

class Freq2WaveOp {  // freq2wave.hpp:32-55 (device-resident)
 public:
  Freq2WaveOp() = default;
  explicit Freq2WaveOp(gs_op* h) : h_(h) { check(gs_op_info(h_, &info_)); }
  ~Freq2WaveOp() {
    if (h_) gs_op_destroy(h_);
  }
  Freq2WaveOp(Freq2WaveOp&& o) noexcept : h_(o.h_), info_(o.info_) { o.h_ = nullptr; }
  Freq2WaveOp& operator=(Freq2WaveOp&& o) noexcept {
    std::swap(h_, o.h_);
    std::swap(info_, o.info_);
    return *this;
  }
  Freq2WaveOp(const Freq2WaveOp&) = delete;
  Freq2WaveOp& operator=(const Freq2WaveOp&) = delete;

  size_t rows() const { return static_cast<size_t>(info_.rows); }
  size_t cols() const { return static_cast<size_t>(info_.cols); }
  bool weighted() const { return info_.weighted != 0; }
  bool uniform_fast() const { return info_.uniform_fast != 0; }
  double uniform_epsilon() const { return info_.uniform_epsilon; }
  int dim() const { return info_.dim; }
  gs_op* handle() const { return h_; }

  // Dx / Lx / Rx (axis 0) or Dy / Ly / Ry (axis 1); L, R column-major M x p
  struct Factors {
    cvec D, L, R;
  };
  Factors factors(int axis) const {
    Factors f;
    const size_t M = rows(), p = static_cast<size_t>(info_.family_p);
    f.D.resize(M);
    if (p >= 2) {
      f.L.resize(M * p);
      f.R.resize(M * p);
    }
    check(gs_op_export_factors(h_, 0, axis, reinterpret_cast<double*>(f.D.data()),
                               p >= 2 ? reinterpret_cast<double*>(f.L.data()) : nullptr,
                               p >= 2 ? reinterpret_cast<double*>(f.R.data()) : nullptr));
    return f;
  }

 private:
  gs_op* h_ = nullptr;
  gs_op_info_t info_{};
};

// freq2wave.cpp:86-193
inline Freq2WaveOp freq2wave(const SamplingSet& samples, Family family, int J,
                             const Freq2WaveOptions& opt = {}) {
  gs_op_desc d{};
  d.dim = samples.dim;
  d.family_p = family_p(family);
  d.J = J;
  d.M = static_cast<int64_t>(samples.size());
  d.batch = 1;
  d.coords = samples.coords.data();
  d.weights = opt.weights.empty() ? nullptr : opt.weights.data();
  if (!opt.weights.empty() && opt.weights.size() != samples.size())
    throw ShapeError("weight count does not match sample count");
  d.bandwidth = opt.bandwidth ? *opt.bandwidth : std::numeric_limits<double>::quiet_NaN();
  d.sigma = opt.sigma;
  d.w = opt.w;
  d.boundary_depth = opt.boundary_depth;
  d.product_terms = opt.product_terms;
  d.allow_uniform_fast_path = opt.allow_uniform_fast_path ? 1 : 0;
  d.allow_tensor_route = opt.allow_tensor_route ? 1 : 0;
  d.device = opt.device;
  gs_op* h = nullptr;
  check(gs_op_create(&d, &h));
  return Freq2WaveOp(h);
}

// freq2wave.cpp:215-303
inline cvec apply_forward(const Freq2WaveOp& op, std::span<const cd> coeffs) {
  cvec out(op.rows());
  check(gs_apply_forward(op.handle(), reinterpret_cast<const double*>(coeffs.data()),
                         static_cast<int64_t>(coeffs.size()), reinterpret_cast<double*>(out.data()), nullptr));
  return out;
}

// freq2wave.cpp:305-387
inline cvec apply_adjoint(const Freq2WaveOp& op, std::span<const cd> samples_vec) {
  cvec out(op.cols());
  check(gs_apply_adjoint(op.handle(), reinterpret_cast<const double*>(samples_vec.data()),
                         static_cast<int64_t>(samples_vec.size()), reinterpret_cast<double*>(out.data()), nullptr));
  return out;
}

struct SolveOptions {  // solver.hpp:10-14
  int max_iterations = 0;
  double tolerance = 1e-10;
  std::optional<cvec> initial_guess;
};

struct SolveStats {  // solver.hpp:16-22
  int iterations = 0;
  double residual = 0.0;
  std::vector<double> history;
  bool converged = false;
};

// solver.cpp:19-91, resident on the GPU
inline std::pair<cvec, SolveStats> solve_least_squares(const Freq2WaveOp& op, std::span<const cd> samples,
                                                       const SolveOptions& options = {}) {
  if (samples.size() != op.rows()) throw ShapeError("sample vector length mismatch");
  if (options.tolerance <= 0) throw DomainError("tolerance must be positive");
  const int max_iter = options.max_iterations > 0 ? options.max_iterations : 2 * static_cast<int>(op.cols());
  if (options.initial_guess && options.initial_guess->size() != op.cols())
    throw ShapeError("initial guess length mismatch");
  cvec x(op.cols());
  std::vector<double> hist(static_cast<size_t>(max_iter) + 1);
  gs_solve_stats st{};
  check(gs_solve_least_squares(op.handle(), reinterpret_cast<const double*>(samples.data()),
                               static_cast<int64_t>(samples.size()),
                               options.initial_guess ? reinterpret_cast<const double*>(options.initial_guess->data())
                                                     : nullptr,
                               options.max_iterations, options.tolerance, reinterpret_cast<double*>(x.data()), &st,
                               hist.data(), nullptr));
  SolveStats stats;
  stats.iterations = st.iterations;
  stats.residual = st.residual;
  stats.converged = st.converged != 0;
  stats.history.assign(hist.begin(), hist.begin() + st.iterations + 1);
  return {std::move(x), std::move(stats)};
}

}  // namespace gs
