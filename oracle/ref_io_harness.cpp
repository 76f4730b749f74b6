// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// C-ABI harness around the UNMODIFIED reference report writers
// (proj/src/io.cpp, proj/src/cost_model.cpp, proj/src/grid.cpp), built by
// oracle/Makefile into oracle/_ref/libanisocg_io_ref.so. tests/test_report.py
// compares the B200 build's io.hpp output with these byte for byte.
#include <cstring>
#include <sstream>
#include <string>

#include "anisocg/grid.hpp"
#include "anisocg/io.hpp"
#include "anisocg/solver.hpp"

using namespace anisocg;

namespace {
long emit(const std::string& s, char* out, long cap) {
    const long n = static_cast<long>(s.size());
    if (out && cap >= n) std::memcpy(out, s.data(), s.size());
    return n;
}
}  // namespace

extern "C" {

long ref_residual_csv(const double* h, int n, char* out, long cap) {
    SolveResult r;
    r.residual_history.assign(h, h + n);
    std::ostringstream os;
    io::write_residual_csv(os, r);
    return emit(os.str(), out, cap);
}

long ref_cost_model_csv(char* out, long cap) {
    std::ostringstream os;
    io::write_cost_model_csv(os);
    return emit(os.str(), out, cap);
}

long ref_geometry_csv(int m, int sphere, double extent, char* out, long cap) {
    const PanelGeometry g = sphere ? build_cubed_sphere_panel(m) : build_planar_panel(m, extent);
    std::ostringstream os;
    io::write_geometry_csv(os, g);
    return emit(os.str(), out, cap);
}

long ref_dump_field(int m, int n_z, int horizontal, int single, const void* data, char* out,
                    long cap) {
    std::ostringstream os;
    const Layout L = horizontal ? Layout::HorizontalContiguous : Layout::VerticalContiguous;
    if (single) {
        Field3D<float> f(m, n_z, L);
        std::memcpy(f.data(), data, f.size() * sizeof(float));
        io::dump_field(os, f);
    } else {
        Field3D<double> f(m, n_z, L);
        std::memcpy(f.data(), data, f.size() * sizeof(double));
        io::dump_field(os, f);
    }
    return emit(os.str(), out, cap);
}

}  // extern "C"
