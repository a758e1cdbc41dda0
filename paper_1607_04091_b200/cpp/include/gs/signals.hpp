// gs/signals.hpp -- drop-in for the reference's include/gs/signals.hpp
// (signals.cpp:11-42; the demo signal of the reconstruction front end).
#pragma once

#include <cmath>
#include <numbers>

#include "gs/nufft.hpp"

namespace gs {

inline double truncated_cosine(double x) {
    if (x >= -0.5 && x < 0.0) return std::cos(2.0 * std::numbers::pi * x);
    return 0.0;
}

inline cd truncated_cosine_transform(double xi) {
    cd out;
    detail::check_inputs(gs_truncated_cosine(1, &xi, reinterpret_cast<double*>(&out)));
    return out;
}

inline cvec truncated_cosine_transform(const SamplingSet& samples) {
    if (samples.dim != 1) throw ShapeError("truncated cosine samples are 1D only");
    cvec out(samples.size());
    detail::check_inputs(gs_truncated_cosine(static_cast<int64_t>(out.size()), samples.coords.data(),
                                             reinterpret_cast<double*>(out.data())));
    return out;
}

}  // namespace gs
