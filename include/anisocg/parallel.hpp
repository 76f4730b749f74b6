#pragma once
// Host-side fixed-shape summation (drop-in for the reference's
// include/anisocg/parallel.hpp: pairwise_sum, parallel.hpp:11-20). The device
// reductions reproduce the same tree (acg_kernels.cu k_tree*);
// this header serves host callers such as grid checks and the reference's
// own unit tests.

#include <cstddef>

namespace anisocg {

// Runs of up to 8 values are summed left to right; longer runs split at
// n / 2 and the two halves' sums are added (a tree fixed by n alone).
template <typename T>
T pairwise_sum(const T* v, std::size_t n) {
    if (n > 8) {
        const std::size_t left = n / 2;
        const T a = pairwise_sum(v, left);
        const T b = pairwise_sum(v + left, n - left);
        return a + b;
    }
    T acc = T(0);
    for (const T* e = v; e != v + n; ++e) acc += *e;
    return acc;
}

}  // namespace anisocg
