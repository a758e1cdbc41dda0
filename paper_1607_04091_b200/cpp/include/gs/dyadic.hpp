// gs/dyadic.hpp -- drop-in for the reference's include/gs/dyadic.hpp
// (dyadic.cpp:14-231): dyadic-grid tables of the scaling / edge functions and
// the weval reconstruction evaluation, computed on the device.
#pragma once

#include <span>
#include <vector>

#include "gs/scaling.hpp"

namespace gs {

struct FunctionTable {
    Family family;
    int resolution;
    long long support_begin;
    std::vector<double> values;

    double value_at(long long numerator) const {
        long long idx = numerator - (support_begin << resolution);
        if (idx < 0 || idx >= static_cast<long long>(values.size())) return 0.0;
        return values[static_cast<size_t>(idx)];
    }
};

inline FunctionTable evaluate_scaling_dyadic(const ScalingFamily& fam, int R) {
    int64_t len = 0, sb = 0;
    detail::check(gs_scaling_dyadic(fam.p, R, nullptr, &len, &sb, nullptr));
    FunctionTable t{fam.name, R, sb, std::vector<double>(static_cast<size_t>(len))};
    detail::check(gs_scaling_dyadic(fam.p, R, t.values.data(), &len, &sb, nullptr));
    return t;
}

inline std::vector<FunctionTable> evaluate_boundary_dyadic(const ScalingFamily& fam, Side side, int R) {
    if (fam.p < 2) throw DomainError("boundary functions require p >= 2");
    std::vector<FunctionTable> out;
    for (int k = 0; k < fam.p; ++k) {
        int64_t len = 0, sb = 0;
        detail::check(gs_boundary_dyadic(fam.p, side == Side::left ? 1 : 0, R, k, nullptr, &len, &sb, nullptr));
        FunctionTable t{fam.name, R, sb, std::vector<double>(static_cast<size_t>(len))};
        detail::check(gs_boundary_dyadic(fam.p, side == Side::left ? 1 : 0, R, k, t.values.data(), &len, &sb, nullptr));
        out.push_back(std::move(t));
    }
    return out;
}

struct ReconstructionEvaluation {
    int resolution;
    int dim;
    std::vector<double> values;

    size_t points_per_axis() const { return (static_cast<size_t>(1) << resolution) + 1; }
};

inline ReconstructionEvaluation weval_1d(std::span<const double> coeffs, const ScalingFamily& fam, int J, int R) {
    ReconstructionEvaluation e{R, 1, std::vector<double>(R >= 0 && R < 31 ? (size_t(1) << R) + 1 : 0)};
    detail::check(gs_weval(1, fam.p, J, R, coeffs.data(), static_cast<int64_t>(coeffs.size()), e.values.data(), nullptr));
    return e;
}

inline ReconstructionEvaluation weval_2d(std::span<const double> coeffs, const ScalingFamily& fam, int J, int R) {
    const size_t g = R >= 0 && R < 16 ? (size_t(1) << R) + 1 : 0;
    ReconstructionEvaluation e{R, 2, std::vector<double>(g * g)};
    detail::check(gs_weval(2, fam.p, J, R, coeffs.data(), static_cast<int64_t>(coeffs.size()), e.values.data(), nullptr));
    return e;
}

}  // namespace gs
