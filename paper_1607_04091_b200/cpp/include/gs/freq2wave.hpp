// gs/freq2wave.hpp -- drop-in for the reference's include/gs/freq2wave.hpp
// (freq2wave.cpp:86-450).  The operator state lives on the B200 (a gs_op
// handle: factors, Kaiser-Bessel tables, sorted bins, workspaces); the
// public fields the reference's callers and tests read (Dx, Lx, ...,
// uniform_fast, zeta_x, sqrt_weights) are host copies filled at construction
// from the device-built factors (gs_op_export_factors).  plan_x / plan_y /
// plan_2d stay empty: the device operator owns its gridding state (the
// lower-level NfftPlan is available separately, gs/nufft.hpp).
#pragma once

#include <Eigen/Dense>
#include <cmath>
#include <limits>
#include <memory>
#include <optional>
#include <span>
#include <vector>

#include "gs/fourier.hpp"
#include "gs/nufft.hpp"
#include "gs/scaling.hpp"

namespace gs {

struct Freq2WaveOptions {
    std::optional<double> bandwidth;
    std::vector<double> weights;
    double sigma = 2.0;
    int w = 6;
    int boundary_depth = kDefaultBoundaryDepth;
    int product_terms = kDefaultProductTerms;
    bool allow_uniform_fast_path = true;
    // B200 additions (defaults keep the reference's routes)
    bool allow_tensor_route = false;  // exact T_x (x) T_y route for uniform 2D grids
    bool exact_ndft = false;          // 1D non-uniform: direct NDFT core instead of the KB NFFT
    int device = 0;
};

struct Freq2WaveOp {
    int dim = 1;
    ScalingFamily family;
    int J = 0;
    long long n = 0;
    SamplingSet samples;
    std::vector<double> sqrt_weights;

    std::vector<double> zeta_x, zeta_y;
    Eigen::VectorXcd Dx, Dy;
    Eigen::MatrixXcd Lx, Rx, Ly, Ry;

    std::optional<NfftPlan> plan_x, plan_y, plan_2d;
    bool uniform_fast = false;
    double uniform_epsilon = 0.0;

    size_t rows() const { return samples.size(); }
    size_t cols() const {
        return dim == 1 ? static_cast<size_t>(n) : static_cast<size_t>(n) * static_cast<size_t>(n);
    }
    bool weighted() const { return !sqrt_weights.empty(); }

    // the device operator (B200 addition)
    gs_op* handle() const { return h_.get(); }
    std::shared_ptr<gs_op> h_;
};

inline Freq2WaveOp freq2wave(const SamplingSet& samples, Family family, int J, const Freq2WaveOptions& options = {}) {
    Freq2WaveOp op;
    op.family = ScalingFamily::make(family);
    op.dim = samples.dim;
    op.J = J;
    op.samples = samples;
    // the checks that precede the weight-count check in freq2wave.cpp:93-108
    // (the library repeats all of them, in the same order)
    if (op.dim != 1 && op.dim != 2) throw DomainError("sampling set must be 1D or 2D");
    if (samples.size() == 0) throw ShapeError("empty sampling set");
    if (J < 0 || J > 24) throw DomainError("scale J out of range");
    if ((1LL << J) < 2 * op.family.p) throw DomainError("scale too small: 2^J must be >= 2p");
    for (double v : samples.coords)
        if (!std::isfinite(v)) throw DomainError("non-finite frequency");
    const size_t M = samples.size();
    if (!options.weights.empty() && options.weights.size() != M)
        throw ShapeError("weight count does not match sample count");
    gs_op_desc d{};
    d.dim = samples.dim;
    d.family_p = op.family.p;
    d.J = J;
    d.M = static_cast<int64_t>(M);
    d.batch = 1;
    d.coords = samples.coords.data();
    d.weights = options.weights.empty() ? nullptr : options.weights.data();
    d.bandwidth = options.bandwidth ? *options.bandwidth : std::numeric_limits<double>::quiet_NaN();
    d.sigma = options.sigma;
    d.w = options.w;
    d.boundary_depth = options.boundary_depth;
    d.product_terms = options.product_terms;
    d.allow_uniform_fast_path = options.allow_uniform_fast_path ? 1 : 0;
    d.allow_tensor_route = options.allow_tensor_route ? 1 : 0;
    d.exact_ndft = options.exact_ndft ? 1 : 0;
    d.device = options.device;
    gs_op* h = nullptr;
    detail::check(gs_op_create(&d, &h));
    op.h_ = std::shared_ptr<gs_op>(h, [](gs_op* p) { gs_op_destroy(p); });
    gs_op_info_t info{};
    detail::check(gs_op_info(h, &info));
    op.n = 1LL << J;
    op.uniform_fast = info.uniform_fast != 0;
    op.uniform_epsilon = info.uniform_epsilon;
    if (!options.weights.empty()) {
        op.sqrt_weights.resize(M);
        for (size_t m = 0; m < M; ++m) op.sqrt_weights[m] = std::sqrt(options.weights[m]);
    }
    op.zeta_x.resize(M);
    for (size_t m = 0; m < M; ++m) op.zeta_x[m] = std::ldexp(samples.x(m), -J);
    if (op.dim == 2) {
        op.zeta_y.resize(M);
        for (size_t m = 0; m < M; ++m) op.zeta_y[m] = std::ldexp(samples.y(m), -J);
    }
    const int p = op.family.p;
    for (int axis = 0; axis < op.dim; ++axis) {
        Eigen::VectorXcd D(static_cast<long>(M));
        Eigen::MatrixXcd L, R;
        if (p >= 2) {
            L = Eigen::MatrixXcd(static_cast<long>(M), p);
            R = Eigen::MatrixXcd(static_cast<long>(M), p);
        }
        detail::check(gs_op_export_factors(h, 0, axis, reinterpret_cast<double*>(D.data()),
                                           p >= 2 ? reinterpret_cast<double*>(L.data()) : nullptr,
                                           p >= 2 ? reinterpret_cast<double*>(R.data()) : nullptr));
        (axis == 0 ? op.Dx : op.Dy) = std::move(D);
        (axis == 0 ? op.Lx : op.Ly) = std::move(L);
        (axis == 0 ? op.Rx : op.Ry) = std::move(R);
    }
    return op;
}

inline cvec apply_forward(const Freq2WaveOp& op, std::span<const cd> coeffs) {
    cvec out(op.rows());
    detail::check(gs_apply_forward(op.handle(), detail::dp(coeffs), static_cast<int64_t>(coeffs.size()),
                                   detail::dp(out), nullptr));
    return out;
}

inline cvec apply_adjoint(const Freq2WaveOp& op, std::span<const cd> samples_vec) {
    cvec out(op.cols());
    detail::check(gs_apply_adjoint(op.handle(), detail::dp(samples_vec), static_cast<int64_t>(samples_vec.size()),
                                   detail::dp(out), nullptr));
    return out;
}

// freq2wave.cpp:420-450: assembled on the device from the transform formulas
inline Eigen::MatrixXcd densify(const Freq2WaveOp& op, size_t entry_cap = size_t(1) << 24) {
    if (op.rows() * op.cols() > entry_cap) throw DomainError("densify: matrix exceeds the entry cap");
    Eigen::MatrixXcd out(static_cast<long>(op.rows()), static_cast<long>(op.cols()));
    detail::check(gs_densify(op.dim, op.family.p, op.J, static_cast<int64_t>(op.rows()), op.samples.coords.data(),
                             op.weighted() ? op.sqrt_weights.data() : nullptr, static_cast<int64_t>(entry_cap),
                             reinterpret_cast<double*>(out.data()), nullptr));
    return out;
}

}  // namespace gs
