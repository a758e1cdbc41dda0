// gs/weights.hpp -- drop-in for the reference's include/gs/weights.hpp
// (weights.cpp:94-176): Voronoi density-compensation weights and the
// density report, computed by the library's exact fast Voronoi
// (csrc/host_inputs.cpp, multi-threaded host code -- the weights are an input).
#pragma once

#include <span>
#include <thread>
#include <vector>

#include "gs/nufft.hpp"

namespace gs {

struct WeightSet {
    std::vector<double> mu;
};

struct DensityReport {
    double delta_raw;
    double delta_scaled;
    bool satisfies_quarter_bound;
};

namespace detail {
inline int host_threads() { return static_cast<int>(std::max(1u, std::thread::hardware_concurrency())); }
inline WeightSet voronoi(int dim, std::span<const double> c, double K) {
    WeightSet w;
    w.mu.resize(c.size() / static_cast<size_t>(dim));
    check_inputs(gs_voronoi_weights(dim, static_cast<int64_t>(w.mu.size()), c.data(), K, w.mu.data(),
                                    host_threads()));
    return w;
}
}  // namespace detail

inline WeightSet voronoi_weights_1d(std::span<const double> points, double K) { return detail::voronoi(1, points, K); }
inline WeightSet voronoi_weights_2d(std::span<const double> xy, double K) {
    if (xy.size() % 2 != 0) throw ShapeError("2D points must be interleaved pairs");
    return detail::voronoi(2, xy, K);
}
inline WeightSet voronoi_weights(const SamplingSet& samples, double K) {
    return samples.dim == 1 ? voronoi_weights_1d(samples.coords, K) : voronoi_weights_2d(samples.coords, K);
}

inline DensityReport density(const SamplingSet& samples, double K) {  // weights.cpp:135-176
    DensityReport r{};
    detail::check_inputs(gs_density(samples.dim, static_cast<int64_t>(samples.size()), samples.coords.data(), K,
                                    &r.delta_raw, detail::host_threads()));
    r.delta_scaled = r.delta_raw / 2.0;
    r.satisfies_quarter_bound = (r.delta_scaled / (2.0 * K)) < 0.25;
    return r;
}

}  // namespace gs
