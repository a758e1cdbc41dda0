// gs/nufft.hpp -- drop-in for the reference's include/gs/nufft.hpp: the direct
// NDFT, the Kaiser-Bessel NfftPlan and the uniform-grid reduction
// (nufft.cpp:74-459), all executed on the B200 through libgs_b200.so.
// Vectors stay std::vector<std::complex<double>> on the host; every call
// copies in and out (device-resident use goes through the C-ABI directly).
#pragma once

#include <array>
#include <complex>
#include <memory>
#include <span>
#include <utility>
#include <vector>

#include "gs/error.hpp"

namespace gs {

using cd = std::complex<double>;
using cvec = std::vector<cd>;

struct SamplingSet {
    int dim = 1;
    std::vector<double> coords;

    size_t size() const { return coords.size() / static_cast<size_t>(dim); }
    double x(size_t m) const { return coords[m * static_cast<size_t>(dim)]; }
    double y(size_t m) const { return coords[m * static_cast<size_t>(dim) + 1]; }
};

namespace detail {
inline const double* dp(std::span<const cd> v) { return reinterpret_cast<const double*>(v.data()); }
inline double* dp(cvec& v) { return reinterpret_cast<double*>(v.data()); }
inline size_t grid_len(int dim, const std::array<int, 2>& N) {
    return static_cast<size_t>(N[0]) * static_cast<size_t>(dim == 2 ? N[1] : 1);
}
}  // namespace detail

inline cvec ndft_forward(int dim, const std::array<int, 2>& N, std::span<const double> points,
                         std::span<const cd> grid) {
    const int64_t M = dim > 0 ? static_cast<int64_t>(points.size() / static_cast<size_t>(dim)) : 0;
    if (dim == 1 || dim == 2) {  // check_points (nufft.cpp:57-66): range, then size
        for (double v : points)
            if (!(v >= -0.5 && v < 0.5)) throw DomainError("scaled point outside [-1/2, 1/2)");
        if (points.empty() || points.size() % static_cast<size_t>(dim) != 0)
            throw ShapeError("point array size is not a multiple of dim");
    }
    cvec out(static_cast<size_t>(M));
    detail::check(gs_ndft_forward(dim, N.data(), points.data(), M, detail::dp(grid),
                                  static_cast<int64_t>(grid.size()), detail::dp(out), nullptr));
    return out;
}

inline cvec ndft_adjoint(int dim, const std::array<int, 2>& N, std::span<const double> points,
                         std::span<const cd> samples) {
    const int64_t M = dim > 0 ? static_cast<int64_t>(points.size() / static_cast<size_t>(dim)) : 0;
    if (dim == 1 || dim == 2) {
        for (double v : points)
            if (!(v >= -0.5 && v < 0.5)) throw DomainError("scaled point outside [-1/2, 1/2)");
        if (points.empty() || points.size() % static_cast<size_t>(dim) != 0)
            throw ShapeError("point array size is not a multiple of dim");
    }
    cvec out(detail::grid_len(dim, N));
    detail::check(gs_ndft_adjoint(dim, N.data(), points.data(), M, detail::dp(samples),
                                  static_cast<int64_t>(samples.size()), detail::dp(out), nullptr));
    return out;
}

// nufft.hpp:36-62: move-only handle to the device plan
class NfftPlan {
  public:
    NfftPlan(int dim, const std::array<int, 2>& N, std::span<const double> points, double sigma, int w,
             int device = 0) {
        const int64_t M = (dim == 1 || dim == 2) ? static_cast<int64_t>(points.size() / static_cast<size_t>(dim)) : 0;
        gs_nfft_plan* h = nullptr;
        detail::check(gs_nfft_plan_create(dim, N.data(), points.data(), M, sigma, w, device, &h));
        h_.reset(h);
    }
    NfftPlan(NfftPlan&&) noexcept = default;
    NfftPlan& operator=(NfftPlan&&) noexcept = default;
    NfftPlan(const NfftPlan&) = delete;
    NfftPlan& operator=(const NfftPlan&) = delete;

    int dim() const { return info().dim; }
    size_t points_count() const { return static_cast<size_t>(info().points); }
    size_t grid_size() const { return static_cast<size_t>(info().grid); }
    int oversampled_length(int axis) const { return info().nov[axis]; }

    cvec forward(std::span<const cd> grid) const {
        cvec out(points_count());
        detail::check(gs_nfft_plan_forward(h_.get(), detail::dp(grid), static_cast<int64_t>(grid.size()),
                                           detail::dp(out), nullptr));
        return out;
    }
    cvec adjoint(std::span<const cd> samples) const {
        cvec out(grid_size());
        detail::check(gs_nfft_plan_adjoint(h_.get(), detail::dp(samples), static_cast<int64_t>(samples.size()),
                                           detail::dp(out), nullptr));
        return out;
    }
    gs_nfft_plan* handle() const { return h_.get(); }

  private:
    struct Info {
        int dim;
        int64_t points, grid;
        int nov[2];
    };
    Info info() const {
        Info i{};
        detail::check(gs_nfft_plan_info(h_.get(), &i.dim, &i.points, &i.grid, i.nov));
        return i;
    }
    struct Del {
        void operator()(gs_nfft_plan* p) const { gs_nfft_plan_destroy(p); }
    };
    std::unique_ptr<gs_nfft_plan, Del> h_;
};

inline NfftPlan plan_nfft(int dim, const std::array<int, 2>& N, std::span<const double> points,
                          double sigma = 2.0, int w = 6) {
    return NfftPlan(dim, N, points, sigma, w);
}
inline cvec nfft_forward(const NfftPlan& plan, std::span<const cd> grid) { return plan.forward(grid); }
inline cvec nfft_adjoint(const NfftPlan& plan, std::span<const cd> samples) { return plan.adjoint(samples); }

inline cvec uniform_ndft_fft(std::span<const cd> x, long long M, double epsilon, long long N) {
    cvec out(static_cast<size_t>(M > 0 ? M : 0));
    detail::check(gs_uniform_ndft_fft(detail::dp(x), static_cast<int64_t>(x.size()), M, epsilon, N,
                                      detail::dp(out), nullptr));
    return out;
}

inline cvec uniform_ndft_adjoint_fft(std::span<const cd> samples, double epsilon, long long N) {
    cvec out(static_cast<size_t>(N > 0 ? N : 0));
    detail::check(gs_uniform_ndft_adjoint_fft(detail::dp(samples), static_cast<int64_t>(samples.size()), epsilon,
                                              N, detail::dp(out), nullptr));
    return out;
}

}  // namespace gs
