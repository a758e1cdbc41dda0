// gs/scaling.hpp -- drop-in for the reference's include/gs/scaling.hpp
// (Family, ScalingFamily, BoundaryFilterSet; scaling.cpp:16-75).  The filter
// and boundary tables are served by libgs_b200.so (the same constants as
// family_tables.cpp, csrc/family_data.h).
#pragma once

#include <Eigen/Dense>
#include <array>
#include <cmath>
#include <map>
#include <mutex>
#include <string>
#include <string_view>
#include <vector>

#include "gs/error.hpp"

namespace gs {

enum class Family { haar, db2, db3, db4, db5, db6, db7, db8 };

inline Family family_from_string(std::string_view name) {  // scaling.cpp:19-25
    static constexpr std::array<std::string_view, 8> names = {"haar", "db2", "db3", "db4",
                                                              "db5",  "db6", "db7", "db8"};
    for (size_t i = 0; i < names.size(); ++i)
        if (name == names[i]) return static_cast<Family>(i);
    if (name == "db1") return Family::haar;
    throw DomainError("unsupported family: " + std::string(name));
}

inline std::string_view family_name(Family f) {
    static constexpr std::array<std::string_view, 8> names = {"haar", "db2", "db3", "db4",
                                                              "db5",  "db6", "db7", "db8"};
    return names[static_cast<size_t>(f)];
}

struct ScalingFamily {
    Family name = Family::haar;
    int p = 1;
    std::vector<double> filter;

    double tap(int k) const {
        if (k < -p + 1 || k > p) return 0.0;
        return filter[static_cast<size_t>(k + p - 1)];
    }

    static ScalingFamily make(Family f) {  // scaling.cpp:29-38
        int p = (f == Family::haar) ? 1 : static_cast<int>(f) + 1;
        ScalingFamily fam;
        fam.name = f;
        fam.p = p;
        fam.filter.resize(static_cast<size_t>(2 * p));
        detail::check(gs_family_filter(p, fam.filter.data()));
        return fam;
    }
};

inline std::vector<double> filter_coefficients(Family f) { return ScalingFamily::make(f).filter; }

enum class Side { left, right };

struct BoundaryFilterSet {
    Side side;
    int p;
    Eigen::MatrixXd H;
    Eigen::MatrixXd h;
    Eigen::MatrixXd U;
    Eigen::MatrixXd V;
    Eigen::MatrixXd integer_values;
};

// cached per (family, side) like scaling.cpp:42-75; DomainError for haar
inline const BoundaryFilterSet& boundary_filters(Family f, Side side) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, BoundaryFilterSet> cache;
    const int p = (f == Family::haar) ? 1 : static_cast<int>(f) + 1;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(p, side == Side::left ? 0 : 1);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    std::vector<double> H(static_cast<size_t>(p * p)), h(static_cast<size_t>(p * (2 * p - 1))),
        iv(static_cast<size_t>(p * 2 * p));
    detail::check(gs_boundary_filter_set(p, side == Side::left ? 1 : 0, H.data(), h.data(), iv.data()));
    BoundaryFilterSet bf{side, p, Eigen::MatrixXd(p, p), Eigen::MatrixXd(p, 2 * p - 1), Eigen::MatrixXd(p, p),
                         Eigen::MatrixXd(p, 2 * p - 1), Eigen::MatrixXd(p, 2 * p)};
    const double r2 = std::sqrt(2.0);
    for (int i = 0; i < p; ++i) {
        for (int j = 0; j < p; ++j) {
            bf.H(i, j) = H[static_cast<size_t>(i * p + j)];
            bf.U(i, j) = bf.H(i, j) / r2;
        }
        for (int j = 0; j < 2 * p - 1; ++j) {
            bf.h(i, j) = h[static_cast<size_t>(i * (2 * p - 1) + j)];
            bf.V(i, j) = bf.h(i, j) / r2;
        }
        for (int j = 0; j < 2 * p; ++j) bf.integer_values(i, j) = iv[static_cast<size_t>(i * 2 * p + j)];
    }
    return cache.emplace(key, std::move(bf)).first->second;
}

}  // namespace gs
