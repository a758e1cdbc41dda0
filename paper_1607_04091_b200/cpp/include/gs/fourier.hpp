// gs/fourier.hpp -- drop-in for the reference's include/gs/fourier.hpp
// (fourier.cpp:16-130).  Evaluations run on the device through the same
// kernels that build the operator's factors (csrc/factors.cuh).
#pragma once

#include <Eigen/Dense>
#include <cmath>
#include <complex>
#include <numbers>

#include "gs/scaling.hpp"

namespace gs {

inline constexpr int kDefaultProductTerms = 48;
inline constexpr int kDefaultBoundaryDepth = 30;

inline std::complex<double> fourier_scaling(const ScalingFamily& fam, double xi,
                                            int terms = kDefaultProductTerms) {
    std::complex<double> out;
    detail::check(gs_fourier_scaling_eval(fam.p, 1, &xi, terms, reinterpret_cast<double*>(&out), nullptr));
    return out;
}

// 2^{-J/2} e^{-2 pi i k xi / 2^J} phihat(xi / 2^J)  (fourier.cpp:51-58)
inline std::complex<double> fourier_scaling_dilated(const ScalingFamily& fam, int J, long long k, double xi,
                                                    int terms = kDefaultProductTerms) {
    double scaled = std::ldexp(xi, -J);
    return std::exp2(-0.5 * J) *
           std::polar(1.0, -2.0 * std::numbers::pi * static_cast<double>(k) * scaled) *
           fourier_scaling(fam, scaled, terms);
}

inline Eigen::VectorXcd boundary_fourier_at_zero(const ScalingFamily& fam, Side side) {
    if (fam.p < 2) throw DomainError("haar has no boundary corrections (p = 1)");
    std::vector<double> v(static_cast<size_t>(fam.p));
    detail::check(gs_boundary_at_zero(fam.p, side == Side::left ? 1 : 0, v.data()));
    Eigen::VectorXcd out(fam.p);
    for (int i = 0; i < fam.p; ++i) out(i) = v[static_cast<size_t>(i)];
    return out;
}

inline Eigen::VectorXcd fourier_boundary(const ScalingFamily& fam, Side side, double xi,
                                         int depth = kDefaultBoundaryDepth,
                                         int terms = kDefaultProductTerms) {
    if (fam.p < 2) throw DomainError("haar has no boundary corrections (p = 1)");
    std::vector<std::complex<double>> v(static_cast<size_t>(fam.p));
    detail::check(gs_fourier_boundary_eval(fam.p, side == Side::left ? 1 : 0, 1, &xi, depth, terms,
                                           reinterpret_cast<double*>(v.data()), nullptr));
    Eigen::VectorXcd out(fam.p);
    for (int i = 0; i < fam.p; ++i) out(i) = v[static_cast<size_t>(i)];
    return out;
}

inline std::complex<double> fourier_scaling_2d(const ScalingFamily& fam, double xi_x, double xi_y,
                                               int terms = kDefaultProductTerms) {
    return fourier_scaling(fam, xi_x, terms) * fourier_scaling(fam, xi_y, terms);
}

struct BoundaryTransformContext {
    ScalingFamily fam;
    Side side;
    Eigen::MatrixXcd U, V;
    Eigen::VectorXcd v_zero;
};

inline BoundaryTransformContext make_boundary_context(const ScalingFamily& fam, Side side) {
    const BoundaryFilterSet& bf = boundary_filters(fam.name, side);
    BoundaryTransformContext ctx;
    ctx.fam = fam;
    ctx.side = side;
    ctx.U = bf.U.cast<std::complex<double>>();
    ctx.V = bf.V.cast<std::complex<double>>();
    ctx.v_zero = boundary_fourier_at_zero(fam, side);
    return ctx;
}

inline Eigen::VectorXcd fourier_boundary(const BoundaryTransformContext& ctx, double xi,
                                         int depth = kDefaultBoundaryDepth,
                                         int terms = kDefaultProductTerms) {
    return fourier_boundary(ctx.fam, ctx.side, xi, depth, terms);
}

}  // namespace gs
