// gs/solver.hpp -- drop-in for the reference's include/gs/solver.hpp
// (solver.cpp:11-104): CGNR resident on the B200 (gs_solve_least_squares),
// and the dense normal-equations oracle for small instances (host, as in the
// reference: a pivoted LDLT of the Gram matrix with the same rank test).
#pragma once

#include <Eigen/Dense>
#include <algorithm>
#include <cmath>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "gs/freq2wave.hpp"

namespace gs {

struct SolveOptions {
    int max_iterations = 0;
    double tolerance = 1e-10;
    std::optional<cvec> initial_guess;
};

struct SolveStats {
    int iterations = 0;
    double residual = 0.0;
    std::vector<double> history;
    bool converged = false;
};

inline std::pair<cvec, SolveStats> solve_least_squares(const Freq2WaveOp& op, std::span<const cd> samples,
                                                       const SolveOptions& options = {}) {
    if (samples.size() != op.rows()) throw ShapeError("sample vector length mismatch");
    if (!(options.tolerance > 0)) throw DomainError("tolerance must be positive");
    if (options.initial_guess && options.initial_guess->size() != op.cols())
        throw ShapeError("initial guess length mismatch");
    const long long mi = options.max_iterations > 0 ? options.max_iterations : 2LL * static_cast<long long>(op.cols());
    cvec x(op.cols());
    std::vector<double> hist(static_cast<size_t>(std::min<long long>(mi, 1LL << 26)) + 1);
    gs_solve_stats st{};
    detail::check(gs_solve_least_squares(
        op.handle(), detail::dp(samples), static_cast<int64_t>(samples.size()),
        options.initial_guess ? reinterpret_cast<const double*>(options.initial_guess->data()) : nullptr,
        options.max_iterations, options.tolerance, detail::dp(x), &st, hist.data(), nullptr));
    SolveStats stats;
    stats.iterations = st.iterations;
    stats.residual = st.residual;
    stats.converged = st.converged != 0;
    stats.history.assign(hist.begin(), hist.begin() + st.iterations + 1);
    return {std::move(x), std::move(stats)};
}

// solver.cpp:93-104: Gram matrix, LDLT with symmetric diagonal pivoting,
// NumericalError when min d <= 1e-13 max |d|
inline Eigen::VectorXcd dense_lsq_oracle(const Eigen::MatrixXcd& matrix, const Eigen::VectorXcd& rhs) {
    if (matrix.rows() != rhs.size()) throw ShapeError("matrix/rhs size mismatch");
    const long n = static_cast<long>(matrix.cols()), m = static_cast<long>(matrix.rows());
    std::vector<cd> A(static_cast<size_t>(n * n)), b(static_cast<size_t>(n));
    for (long j = 0; j < n; ++j) {
        for (long i = 0; i < n; ++i) {
            cd acc = 0.0;
            for (long k = 0; k < m; ++k) acc += std::conj(matrix(k, i)) * matrix(k, j);
            A[static_cast<size_t>(i * n + j)] = acc;
        }
        cd acc = 0.0;
        for (long k = 0; k < m; ++k) acc += std::conj(matrix(k, j)) * rhs(k);
        b[static_cast<size_t>(j)] = acc;
    }
    auto a = [&](long i, long j) -> cd& { return A[static_cast<size_t>(i * n + j)]; };
    std::vector<long> perm(static_cast<size_t>(n));
    for (long i = 0; i < n; ++i) perm[static_cast<size_t>(i)] = i;
    std::vector<double> d(static_cast<size_t>(n));
    for (long k = 0; k < n; ++k) {
        long best = k;
        for (long i = k + 1; i < n; ++i)
            if (std::abs(a(i, i)) > std::abs(a(best, best))) best = i;
        if (best != k) {
            for (long j = 0; j < n; ++j) std::swap(a(k, j), a(best, j));
            for (long i = 0; i < n; ++i) std::swap(a(i, k), a(i, best));
            std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(best)]);
        }
        const cd dk = a(k, k);
        d[static_cast<size_t>(k)] = dk.real();
        if (dk == cd(0.0)) continue;
        for (long i = k + 1; i < n; ++i) a(i, k) /= dk;
        for (long j = k + 1; j < n; ++j)
            for (long i = j; i < n; ++i) a(i, j) -= a(i, k) * dk * std::conj(a(j, k));
        for (long j = k + 1; j < n; ++j)
            for (long i = k + 1; i < j; ++i) a(i, j) = std::conj(a(j, i));
    }
    double dmax = 0.0, dmin = n ? d[0] : 0.0;
    for (double v : d) {
        dmax = std::max(dmax, std::abs(v));
        dmin = std::min(dmin, v);
    }
    if (n == 0 || dmin <= dmax * 1e-13) throw NumericalError("dense least squares: rank-deficient system");
    std::vector<cd> y(static_cast<size_t>(n));
    for (long i = 0; i < n; ++i) y[static_cast<size_t>(i)] = b[static_cast<size_t>(perm[static_cast<size_t>(i)])];
    for (long i = 0; i < n; ++i)
        for (long k = 0; k < i; ++k) y[static_cast<size_t>(i)] -= a(i, k) * y[static_cast<size_t>(k)];
    for (long i = 0; i < n; ++i) y[static_cast<size_t>(i)] /= a(i, i);
    for (long i = n - 1; i >= 0; --i)
        for (long k = i + 1; k < n; ++k) y[static_cast<size_t>(i)] -= std::conj(a(k, i)) * y[static_cast<size_t>(k)];
    Eigen::VectorXcd x(n);
    for (long i = 0; i < n; ++i) x(perm[static_cast<size_t>(i)]) = y[static_cast<size_t>(i)];
    return x;
}

}  // namespace gs
