#pragma once
// Drop-in for proj/include/anisocg/grid.hpp: host-side setup, computed once per
// problem in double precision (bit-identical to the reference; see
// tests/test_setup.py). Implementation: paper_1302_7193_b200/csrc/host/grid.cpp.
#include <cstddef>
#include <vector>

namespace anisocg {

/// grid.hpp:10-14
struct VerticalGrid {
    int n_z = 0;
    double h_atmos = 0.0;
    std::vector<double> r;  ///< n_z+1 interface radii, r[0] = 1
};

/// r_k = 1 + (k/n_z)^2 h_atmos (grid.cpp:10-24)
VerticalGrid build_graded_vertical_grid(int n_z, double h_atmos);

/// grid.hpp:30-44 — per-cell areas and per-edge couplings of an m x m panel.
class PanelGeometry {
public:
    int m = 0;
    std::vector<double> cell_area;    // m*m, index i*m + j
    std::vector<double> alpha_east;   // (m-1)*m, edge (i,j)-(i+1,j), index i*m + j
    std::vector<double> alpha_north;  // m*(m-1), edge (i,j)-(i,j+1), index i*(m-1) + j
    std::vector<double> alpha_diag;   // m*m

    double area(int i, int j) const { return cell_area[static_cast<std::size_t>(i) * m + j]; }
    double east(int i, int j) const { return alpha_east[static_cast<std::size_t>(i) * m + j]; }
    double north(int i, int j) const {
        return alpha_north[static_cast<std::size_t>(i) * (m - 1) + j];
    }
    double diag(int i, int j) const { return alpha_diag[static_cast<std::size_t>(i) * m + j]; }
};

/// Gnomonic cubed-sphere panel (grid.cpp:88-125)
PanelGeometry build_cubed_sphere_panel(int m);
/// Uniform planar panel (grid.cpp:127-139)
PanelGeometry build_planar_panel(int m, double extent);
/// gamma^2 = lambda2 * area / dz^2 in column order (grid.cpp:141-156)
std::vector<double> anisotropy(const PanelGeometry& geometry, const VerticalGrid& vgrid,
                               double lambda2);

}  // namespace anisocg
