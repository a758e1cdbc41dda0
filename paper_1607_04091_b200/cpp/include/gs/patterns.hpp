// gs/patterns.hpp -- drop-in for the reference's include/gs/patterns.hpp
// (patterns.cpp:14-74; bit-identical doubles, csrc/host_inputs.cpp).
#pragma once

#include <cmath>
#include <cstdint>

#include "gs/nufft.hpp"

namespace gs {

inline SamplingSet gen_grid(long long M, double epsilon, int dim = 1) {
    SamplingSet s;
    s.dim = dim;
    if (M >= 1 && (dim == 1 || dim == 2)) s.coords.resize(static_cast<size_t>(dim == 2 ? 2 * M * M : M));
    detail::check_inputs(gs_gen_grid(M, epsilon, dim, s.coords.data()));
    return s;
}

inline SamplingSet gen_jitter(long long M, double epsilon, double eta, uint64_t seed, int dim = 1) {
    SamplingSet s;
    s.dim = dim;
    if (M >= 1 && (dim == 1 || dim == 2)) s.coords.resize(static_cast<size_t>(dim == 2 ? 2 * M * M : M));
    detail::check_inputs(gs_gen_jitter(M, epsilon, eta, seed, dim, s.coords.data()));
    return s;
}

inline SamplingSet gen_spiral(int turns, double points_per_turn, double K) {
    SamplingSet s;
    s.dim = 2;
    if (turns >= 1 && points_per_turn > 0)
        s.coords.resize(2 * static_cast<size_t>(std::llround(turns * points_per_turn)));
    detail::check_inputs(gs_gen_spiral(turns, points_per_turn, K, s.coords.data()));
    return s;
}

}  // namespace gs
