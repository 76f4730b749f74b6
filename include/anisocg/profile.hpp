#pragma once
// Drop-in for proj/include/anisocg/profile.hpp (host-side, once per problem).
#include <vector>

#include "anisocg/grid.hpp"

namespace anisocg {

/// profile.hpp:18-26 — scaled per-level coefficients a' = a/d, b' = b/d, c' = c/d, d.
struct VerticalProfile {
    int n_z = 0;
    double omega2 = 0.0;
    double lambda2 = 0.0;
    std::vector<double> a_prime, b_prime, c_prime, d;
};

/// profile.cpp:7-48
VerticalProfile build_vertical_profile(const VerticalGrid& vgrid, double omega2, double lambda2);

}  // namespace anisocg
