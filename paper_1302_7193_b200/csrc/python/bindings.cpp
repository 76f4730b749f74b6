// _anisocg: the reference's Python module surface (proj/python/bindings.cpp:77-247)
// over the B200 shim. Fields cross as C-contiguous (m, m, n_z) arrays (the
// vertically contiguous layout, bindings.cpp:1-3); every compute call runs on
// the GPU. Extensions (keyword-only, defaults keep the reference behaviour):
// fp32 contexts, `layout="horizontal"` host arrays ((m, n_z, m), [j, k, i]),
// multi-slab placement, the fused sweeps and the level-1 operations.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <array>
#include <sstream>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "acg.h"
#include "anisocg/csr.hpp"
#include "anisocg/field.hpp"
#include "anisocg/grid.hpp"
#include "anisocg/io.hpp"
#include "anisocg/operator.hpp"
#include "anisocg/profile.hpp"
#include "anisocg/solver.hpp"

namespace py = pybind11;
using namespace anisocg;

namespace {

template <typename T>
using Arr = py::array_t<T, py::array::c_style | py::array::forcecast>;

py::array_t<double> vec(const std::vector<double>& v) {
    py::array_t<double> out(static_cast<py::ssize_t>(v.size()));
    if (!v.empty()) std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(double));
    return out;
}

py::array_t<double> mat(const std::vector<double>& v, py::ssize_t r, py::ssize_t c) {
    py::array_t<double> out({r, c});
    if (!v.empty()) std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(double));
    return out;
}

Layout parse_layout(const std::string& s) {
    if (s == "vertical") return Layout::VerticalContiguous;
    if (s == "horizontal") return Layout::HorizontalContiguous;
    throw std::invalid_argument("layout must be 'vertical' or 'horizontal'");
}

template <typename T>
Field3D<T> to_field(const Arr<T>& a, int m, int n_z, Layout layout) {
    const bool vert = layout == Layout::VerticalContiguous;
    const py::ssize_t s1 = vert ? m : n_z, s2 = vert ? n_z : m;
    if (a.ndim() != 3 || a.shape(0) != m || a.shape(1) != s1 || a.shape(2) != s2)
        throw std::invalid_argument(vert ? "expected a (m, m, n_z) array matching the operator context"
                                         : "expected a (m, n_z, m) array matching the operator context");
    Field3D<T> f(m, n_z, layout);
    std::memcpy(f.data(), a.data(), f.size() * sizeof(T));
    return f;
}

// Zero-copy host edge: numpy buffers go straight to the C ABI's host entry
// points (which upload, relayout on the device and download), with no
// intermediate Field3D copies — at 1024^2 x 128 each such copy is a 1 GB
// memcpy or memset on the host.
template <typename T>
void check_shape(const Arr<T>& a, int m, int n_z, Layout layout) {
    const bool vert = layout == Layout::VerticalContiguous;
    const py::ssize_t s1 = vert ? m : n_z, s2 = vert ? n_z : m;
    if (a.ndim() != 3 || a.shape(0) != m || a.shape(1) != s1 || a.shape(2) != s2)
        throw std::invalid_argument(vert ? "expected a (m, m, n_z) array matching the operator context"
                                         : "expected a (m, n_z, m) array matching the operator context");
}

template <typename T>
py::array_t<T> new_field_array(int m, int n_z, Layout layout) {
    const bool vert = layout == Layout::VerticalContiguous;
    return py::array_t<T>(vert ? std::vector<py::ssize_t>{m, m, n_z}
                               : std::vector<py::ssize_t>{m, n_z, m});
}

// SolveResult from the C ABI result whose histories the library allocated.
SolveResult result_of(acg_solve_result& r) {
    SolveResult res;
    res.iterations = r.iterations;
    res.converged = r.converged != 0;
    res.true_residual = r.true_residual;
    res.residual_history.assign(r.history[0], r.history[0] + r.n_residual);
    res.kappa_history.assign(r.history[1], r.history[1] + r.n_kappa);
    res.alpha_history.assign(r.history[2], r.history[2] + r.n_alpha);
    res.beta_history.assign(r.history[3], r.history[3] + r.n_beta);
    res.timings.spmv = r.timings.spmv;
    res.timings.prec = r.timings.prec;
    res.timings.blas = r.timings.blas;
    res.timings.fused_spmv = r.timings.fused_spmv;
    res.timings.fused_prec = r.timings.fused_prec;
    res.timings.setup = r.timings.setup;
    res.timings.total = r.timings.total;
    acg_solve_result_release(&r);
    return res;
}

template <typename T>
py::array_t<T> to_array(const Field3D<T>& f) {
    const bool vert = f.layout() == Layout::VerticalContiguous;
    const py::ssize_t m = f.m(), n_z = f.n_z();
    py::array_t<T> out(vert ? std::vector<py::ssize_t>{m, m, n_z}
                            : std::vector<py::ssize_t>{m, n_z, m});
    std::memcpy(out.mutable_data(), f.data(), f.size() * sizeof(T));
    return out;
}

acg_placement placement(int slabs, const std::string& math, int device) {
    acg_placement p{};
    p.device = device;
    p.slabs = slabs;
    p.comm = nullptr;
    if (math == "exact")
        p.math = ACG_MATH_EXACT;
    else if (math == "fast")
        p.math = ACG_MATH_FAST;
    else
        throw std::invalid_argument("math must be 'exact' or 'fast'");
    return p;
}

// Cost tables of the paper (Tables 1-2), proj/src/cost_model.cpp:17-32.
std::pair<int, int> cost(const std::string& kernel, const std::string& cache) {
    static const char* names[] = {"spmv",       "prec",     "blas", "interleaved_spmv",
                                  "interleaved_prec", "pcg_total", "interleaved_total"};
    static const int flops[] = {20, 13, 13, 28, 19, 46, 47};
    static const int mem[][3] = {{12, 8, 6},   {12, 8, 5},   {16, 16, 16}, {17, 13, 11},
                                 {16, 12, 9},  {40, 32, 27}, {33, 25, 20}};
    static const char* caches[] = {"none", "matrix_cached", "columns_cached"};
    int ki = -1, ci = -1;
    for (int a = 0; a < 7; ++a)
        if (kernel == names[a]) ki = a;
    for (int a = 0; a < 3; ++a)
        if (cache == caches[a]) ci = a;
    if (ki < 0) throw std::invalid_argument("unknown kernel: " + kernel);
    if (ci < 0) throw std::invalid_argument("unknown cache assumption: " + cache);
    return {flops[ki], mem[ki][ci]};
}

// assemble_csr(ctx, VerticalContiguous) as (row_ptr, col_idx, vals) arrays
// (bindings.cpp:179-193; host utility for the scipy cross-check).
py::tuple csr_arrays(const OperatorContext<double>& ctx) {
    const CsrMatrix<double> A = assemble_csr(ctx, Layout::VerticalContiguous);
    py::array_t<std::int64_t> a(static_cast<py::ssize_t>(A.row_ptr.size()));
    std::memcpy(a.mutable_data(), A.row_ptr.data(), A.row_ptr.size() * sizeof(std::int64_t));
    py::array_t<std::int32_t> b(static_cast<py::ssize_t>(A.col_idx.size()));
    std::memcpy(b.mutable_data(), A.col_idx.data(), A.col_idx.size() * sizeof(std::int32_t));
    return py::make_tuple(a, b, vec(A.vals));
}

template <typename T, typename Cls>
void bind_context(py::module_& mod, const char* name) {
    py::class_<OperatorContext<T>>(mod, name)
        .def(py::init([](const VerticalProfile& p, const PanelGeometry& g, int slabs,
                         const std::string& math, int device) {
                 const acg_placement pl = placement(slabs, math, device);
                 return new OperatorContext<T>(p, g, &pl);
             }),
             py::arg("profile"), py::arg("geometry"), py::kw_only(), py::arg("slabs") = 1,
             py::arg("math") = "exact", py::arg("device") = 0)
        .def_property_readonly("m", &OperatorContext<T>::m)
        .def_property_readonly("n_z", &OperatorContext<T>::n_z)
        .def_property_readonly("_handle", [](const OperatorContext<T>& c) {
            return reinterpret_cast<std::uintptr_t>(c.device());
        })
        .def_property_readonly("info", [](const OperatorContext<T>& c) {
            acg_context_info i{};
            detail::check(acg_context_info_get(c.device(), &i));
            py::dict d;
            d["m"] = i.m;
            d["n_z"] = i.n_z;
            d["dtype"] = i.dtype == ACG_F32 ? "f32" : "f64";
            d["math"] = i.math == ACG_MATH_FAST ? "fast" : "exact";
            d["slabs"] = i.nslabs_total;
            d["exact_tree"] = static_cast<bool>(i.exact_tree);
            d["bytes_per_field"] = i.bytes_per_field_local;
            d["thomas_tmem"] = static_cast<bool>(i.thomas_tmem);
            return d;
        })
        .def(
            "release_scratch",
            [](const OperatorContext<T>& c) { detail::release_scratch(c.device()); },
            "Free the device scratch cached between calls (re-created on demand)");
    (void)sizeof(Cls);
}

template <typename T>
void bind_ops(py::module_& mod) {
    using Ctx = OperatorContext<T>;
    mod.def(
        "apply",
        [](const Ctx& ctx, const Arr<T>& x, int workers, const std::string& layout) {
            (void)workers;
            const Layout L = parse_layout(layout);
            check_shape<T>(x, ctx.m(), ctx.n_z(), L);
            auto y = new_field_array<T>(ctx.m(), ctx.n_z(), L);
            const T* xp = x.data();
            T* yp = y.mutable_data();
            acg_status st;
            {
                py::gil_scoped_release nogil;
                st = acg_apply_host(ctx.device(), detail::layout_of(L), xp, yp);
            }
            detail::check(st);
            return y;
        },
        py::arg("ctx"), py::arg("x"), py::arg("workers") = 1, py::kw_only(),
        py::arg("layout") = "vertical", "y = A x (matrix-free stencil, sm_100a)");
    mod.def(
        "precondition",
        [](const Ctx& ctx, const Arr<T>& y, int workers, const std::string& layout) {
            (void)workers;
            const Layout L = parse_layout(layout);
            check_shape<T>(y, ctx.m(), ctx.n_z(), L);
            auto x = new_field_array<T>(ctx.m(), ctx.n_z(), L);
            const T* yp = y.data();
            T* xp = x.mutable_data();
            acg_status st;
            {
                py::gil_scoped_release nogil;
                st = acg_precondition_host(ctx.device(), detail::layout_of(L), yp, xp);
            }
            detail::check(st);
            return x;
        },
        py::arg("ctx"), py::arg("y"), py::arg("workers") = 1, py::kw_only(),
        py::arg("layout") = "vertical", "x = M^-1 y (per-column Thomas solves, sm_100a)");
    mod.def(
        "solve",
        [](const Ctx& ctx, const Arr<T>& f, py::object u0, double epsilon, double tau,
           int maxiter, const std::string& variant, const std::string& backend, int workers,
           const std::string& layout) {
            const Layout L = parse_layout(layout);
            check_shape<T>(f, ctx.m(), ctx.n_z(), L);
            Arr<T> u0a;
            if (!u0.is_none()) {
                u0a = u0.cast<Arr<T>>();
                check_shape<T>(u0a, ctx.m(), ctx.n_z(), L);
            }
            SolverConfig cfg;
            cfg.epsilon = epsilon;
            cfg.tau = tau;
            cfg.maxiter = maxiter;
            cfg.workers = workers;
            if (variant == "standard")
                cfg.variant = Variant::standard;
            else if (variant == "interleaved")
                cfg.variant = Variant::interleaved;
            else
                throw std::invalid_argument("variant must be 'standard' or 'interleaved'");
            if (backend == "matrix-free")
                cfg.backend = BackendKind::matrix_free;
            else if (backend == "csr")
                cfg.backend = BackendKind::csr;
            else
                throw std::invalid_argument("backend must be 'matrix-free' or 'csr'");
            cfg.validate();  // SolverConfig::validate (solver.hpp:27-35): the reference's messages
            acg_solver_config c{};
            acg_solver_config_default(&c);
            c.epsilon = cfg.epsilon;
            c.tau = cfg.tau;
            c.maxiter = cfg.maxiter;
            c.workers = cfg.workers;
            c.variant = cfg.variant == Variant::interleaved ? ACG_VARIANT_INTERLEAVED
                                                             : ACG_VARIANT_STANDARD;
            c.backend = cfg.backend == BackendKind::csr ? ACG_BACKEND_CSR : ACG_BACKEND_MATRIX_FREE;
            c.record_timings = 1;
            auto u = new_field_array<T>(ctx.m(), ctx.n_z(), L);
            const T* fp = f.data();
            const T* u0p = u0.is_none() ? nullptr : u0a.data();  // NULL: zero start, no upload
            T* up = u.mutable_data();
            acg_solve_result r{};
            acg_status st;
            {
                py::gil_scoped_release nogil;
                st = acg_solve_host(ctx.device(), detail::layout_of(L), fp, u0p, &c, up, &r,
                                    nullptr, nullptr, nullptr, nullptr);
            }
            detail::check(st);
            return py::make_tuple(u, result_of(r));
        },
        py::arg("ctx"), py::arg("f"), py::arg("u0") = py::none(), py::arg("epsilon") = 1e-5,
        py::arg("tau") = 1e-20, py::arg("maxiter") = 500, py::arg("variant") = "interleaved",
        py::arg("backend") = "matrix-free", py::arg("workers") = 1, py::kw_only(),
        py::arg("layout") = "vertical", "Preconditioned CG solve on the GPU; returns (u, SolveResult)");
    mod.def(
        "true_residual",
        [](const Ctx& ctx, const Arr<T>& u, const Arr<T>& f, int workers,
           const std::string& layout) {
            (void)workers;
            const Layout L = parse_layout(layout);
            check_shape<T>(u, ctx.m(), ctx.n_z(), L);
            check_shape<T>(f, ctx.m(), ctx.n_z(), L);
            double out = 0.0;
            const T* up = u.data();
            const T* fp = f.data();
            acg_status st;
            {
                py::gil_scoped_release nogil;
                st = acg_true_residual_host(ctx.device(), detail::layout_of(L), up, fp, &out);
            }
            detail::check(st);
            // nrm2's sqrt in T (field.hpp:172), then widened like the reference binding
            return static_cast<double>(static_cast<T>(out));
        },
        py::arg("ctx"), py::arg("u"), py::arg("f"), py::arg("workers") = 1, py::kw_only(),
        py::arg("layout") = "vertical", "||f - A u|| recomputed from scratch");
    mod.def(
        "interleaved_spmv_kernel",
        [](const Ctx& ctx, const Arr<T>& u, const Arr<T>& p, const Arr<T>& q, const Arr<T>& z,
           double alpha, double beta, const std::string& layout) {
            const Layout L = parse_layout(layout);
            FusedState<T> st(ctx.m(), ctx.n_z(), L);
            st.u = to_field<T>(u, ctx.m(), ctx.n_z(), L);
            st.p = to_field<T>(p, ctx.m(), ctx.n_z(), L);
            st.q = to_field<T>(q, ctx.m(), ctx.n_z(), L);
            st.z = to_field<T>(z, ctx.m(), ctx.n_z(), L);
            st.alpha = static_cast<T>(alpha);
            st.beta = static_cast<T>(beta);
            const T sigma = interleaved_spmv_kernel(ctx, st);
            return py::make_tuple(to_array(st.u), to_array(st.p), to_array(st.q),
                                  static_cast<double>(sigma));
        },
        py::arg("ctx"), py::arg("u"), py::arg("p"), py::arg("q"), py::arg("z"), py::arg("alpha"),
        py::arg("beta"), py::kw_only(), py::arg("layout") = "vertical",
        "Fused sweep (Alg. 2): returns (u, p, q, sigma)");
    mod.def(
        "interleaved_prec_kernel",
        [](const Ctx& ctx, const Arr<T>& r, const Arr<T>& q, double alpha,
           const std::string& layout) {
            const Layout L = parse_layout(layout);
            FusedState<T> st(ctx.m(), ctx.n_z(), L);
            st.r = to_field<T>(r, ctx.m(), ctx.n_z(), L);
            st.q = to_field<T>(q, ctx.m(), ctx.n_z(), L);
            st.alpha = static_cast<T>(alpha);
            const auto rk = interleaved_prec_kernel(ctx, st);
            return py::make_tuple(to_array(st.r), to_array(st.z), static_cast<double>(rk.first),
                                  static_cast<double>(rk.second));
        },
        py::arg("ctx"), py::arg("r"), py::arg("q"), py::arg("alpha"), py::kw_only(),
        py::arg("layout") = "vertical", "Fused sweep (Alg. 3): returns (r, z, r_norm, kappa)");
}

template <typename T>
void bind_blas(py::module_& mod) {
    auto field = [](const Arr<T>& a, const std::string& layout) {
        if (a.ndim() != 3) throw std::invalid_argument("expected a 3-d array");
        const Layout L = parse_layout(layout);
        const int m = static_cast<int>(a.shape(0));
        const int n_z = static_cast<int>(L == Layout::VerticalContiguous ? a.shape(2) : a.shape(1));
        return to_field<T>(a, m, n_z, L);
    };
    mod.def(
        "dot",
        [field](const Arr<T>& x, const Arr<T>& y, const std::string& layout) {
            return static_cast<double>(dot(field(x, layout), field(y, layout)));
        },
        py::arg("x"), py::arg("y"), py::kw_only(), py::arg("layout") = "vertical");
    mod.def(
        "nrm2",
        [field](const Arr<T>& x, const std::string& layout) {
            return static_cast<double>(nrm2(field(x, layout)));
        },
        py::arg("x"), py::kw_only(), py::arg("layout") = "vertical");
    mod.def(
        "axpy",
        [field](double alpha, const Arr<T>& x, const Arr<T>& y, const std::string& layout) {
            auto yf = field(y, layout);
            axpy(static_cast<T>(alpha), field(x, layout), yf);
            return to_array(yf);
        },
        py::arg("alpha"), py::arg("x"), py::arg("y"), py::kw_only(), py::arg("layout") = "vertical");
    mod.def(
        "scal",
        [field](double alpha, const Arr<T>& x, const std::string& layout) {
            auto xf = field(x, layout);
            scal(static_cast<T>(alpha), xf);
            return to_array(xf);
        },
        py::arg("alpha"), py::arg("x"), py::kw_only(), py::arg("layout") = "vertical");
}

}  // namespace

PYBIND11_MODULE(_anisocg, mod) {
    mod.doc() = "B200-native matrix-free PCG solver for strongly anisotropic elliptic equations";

    py::class_<VerticalGrid>(mod, "VerticalGrid")
        .def_readonly("n_z", &VerticalGrid::n_z)
        .def_readonly("h_atmos", &VerticalGrid::h_atmos)
        .def_property_readonly("r", [](const VerticalGrid& g) { return vec(g.r); });

    py::class_<PanelGeometry>(mod, "PanelGeometry")
        .def_readonly("m", &PanelGeometry::m)
        .def_property_readonly("cell_area",
                               [](const PanelGeometry& g) { return mat(g.cell_area, g.m, g.m); })
        .def_property_readonly("alpha_east",
                               [](const PanelGeometry& g) { return mat(g.alpha_east, g.m - 1, g.m); })
        .def_property_readonly("alpha_north",
                               [](const PanelGeometry& g) { return mat(g.alpha_north, g.m, g.m - 1); })
        .def_property_readonly("alpha_diag",
                               [](const PanelGeometry& g) { return mat(g.alpha_diag, g.m, g.m); });

    py::class_<VerticalProfile>(mod, "VerticalProfile")
        .def_readonly("n_z", &VerticalProfile::n_z)
        .def_readonly("omega2", &VerticalProfile::omega2)
        .def_readonly("lambda2", &VerticalProfile::lambda2)
        .def_property_readonly("a_prime", [](const VerticalProfile& p) { return vec(p.a_prime); })
        .def_property_readonly("b_prime", [](const VerticalProfile& p) { return vec(p.b_prime); })
        .def_property_readonly("c_prime", [](const VerticalProfile& p) { return vec(p.c_prime); })
        .def_property_readonly("d", [](const VerticalProfile& p) { return vec(p.d); });

    bind_context<double, int>(mod, "OperatorContext");
    bind_context<float, int>(mod, "OperatorContextF32");

    py::class_<KernelTimings>(mod, "KernelTimings")
        .def_readonly("spmv_s", &KernelTimings::spmv)
        .def_readonly("prec_s", &KernelTimings::prec)
        .def_readonly("blas_s", &KernelTimings::blas)
        .def_readonly("fused_spmv_s", &KernelTimings::fused_spmv)
        .def_readonly("fused_prec_s", &KernelTimings::fused_prec)
        .def_readonly("setup_s", &KernelTimings::setup)
        .def_readonly("total_s", &KernelTimings::total);

    py::class_<SolveResult>(mod, "SolveResult")
        .def_readonly("iterations", &SolveResult::iterations)
        .def_readonly("converged", &SolveResult::converged)
        .def_readonly("true_residual", &SolveResult::true_residual)
        .def_readonly("timings", &SolveResult::timings)
        .def_property_readonly("residual_history",
                               [](const SolveResult& r) { return vec(r.residual_history); })
        .def_property_readonly("kappa_history",
                               [](const SolveResult& r) { return vec(r.kappa_history); })
        .def_property_readonly("alpha_history",
                               [](const SolveResult& r) { return vec(r.alpha_history); })
        .def_property_readonly("beta_history",
                               [](const SolveResult& r) { return vec(r.beta_history); });

    mod.def("vertical_grid", &build_graded_vertical_grid, py::arg("n_z"), py::arg("h_atmos"),
            "Quadratically graded vertical grid on [1, 1 + h_atmos]");
    mod.def("cubed_sphere_panel", &build_cubed_sphere_panel, py::arg("m"),
            "Gnomonic cubed-sphere panel geometry");
    mod.def("planar_panel", &build_planar_panel, py::arg("m"), py::arg("extent"),
            "Uniform planar panel geometry");
    mod.def("vertical_profile", &build_vertical_profile, py::arg("grid"), py::arg("omega2"),
            py::arg("lambda2"), "Scaled vertical coefficients a', b', c', d");
    mod.def(
        "anisotropy",
        [](const PanelGeometry& g, const VerticalGrid& vg, double lambda2) {
            const auto a = anisotropy(g, vg, lambda2);
            py::array_t<double> out({static_cast<py::ssize_t>(g.m), static_cast<py::ssize_t>(g.m),
                                     static_cast<py::ssize_t>(vg.n_z)});
            std::memcpy(out.mutable_data(), a.data(), a.size() * sizeof(double));
            return out;
        },
        py::arg("geometry"), py::arg("grid"), py::arg("lambda2"));

    // fp32 overloads first: pybind tries overloads in order and the context type decides.
    bind_ops<float>(mod);
    bind_ops<double>(mod);
    bind_blas<double>(mod);

    mod.def("assemble_csr", &csr_arrays, py::arg("ctx"),
            "CSR arrays (row_ptr, col_idx, vals) in vertically contiguous row order "
            "(host verification utility)");
    mod.def(
        "cost_model",
        [](const std::string& kernel, const std::string& cache) {
            const auto c = cost(kernel, cache);
            return py::make_tuple(c.first, c.second);
        },
        py::arg("kernel"), py::arg("cache") = "none",
        "(flops, mem_refs) per grid point (paper Tables 1-2)");
    mod.def(
        "random_field",
        [](int m, int n_z, std::uint64_t seed, const std::string& dtype) {
            if (dtype == "float32") {
                Field3D<float> f(m, n_z, Layout::VerticalContiguous);
                fill_random(f, seed);
                return py::object(to_array(f));
            }
            Field3D<double> f(m, n_z, Layout::VerticalContiguous);
            fill_random(f, seed);
            return py::object(to_array(f));
        },
        py::arg("m"), py::arg("n_z"), py::arg("seed") = 42, py::kw_only(),
        py::arg("dtype") = "float64", "The deterministic benchmark right-hand side (GPU generated)");
    // report and wire formats (io.hpp); the text is returned for the caller to write
    mod.def(
        "residual_csv",
        [](py::object r) {
            SolveResult res;
            py::object h = py::hasattr(r, "residual_history") ? r.attr("residual_history") : r;
            const Arr<double> a = h.cast<Arr<double>>();
            res.residual_history.assign(a.data(), a.data() + a.size());
            std::ostringstream os;
            io::write_residual_csv(os, res);
            return os.str();
        },
        py::arg("result"), "io::write_residual_csv as a string (a SolveResult or a history array)");
    mod.def(
        "cost_model_csv",
        [] {
            std::ostringstream os;
            io::write_cost_model_csv(os);
            return os.str();
        },
        "io::write_cost_model_csv as a string");
    mod.def(
        "geometry_csv",
        [](const PanelGeometry& g) {
            std::ostringstream os;
            io::write_geometry_csv(os, g);
            return os.str();
        },
        py::arg("geometry"), "io::write_geometry_csv as a string");
    mod.def(
        "dump_field",
        [](py::array a, const std::string& layout) {
            const Layout L = parse_layout(layout);
            const bool vert = L == Layout::VerticalContiguous;
            if (a.ndim() != 3) throw std::invalid_argument("expected a 3D field array");
            const int m = static_cast<int>(a.shape(0));
            const int n_z = static_cast<int>(vert ? a.shape(2) : a.shape(1));
            std::ostringstream os;
            if (py::isinstance<py::array_t<float>>(a)) {
                io::dump_field(os, to_field<float>(a.cast<Arr<float>>(), m, n_z, L));
            } else {
                io::dump_field(os, to_field<double>(a.cast<Arr<double>>(), m, n_z, L));
            }
            return py::bytes(os.str());
        },
        py::arg("field"), py::kw_only(), py::arg("layout") = "vertical",
        "io::dump_field: text header + raw little-endian values (bytes)");
    mod.def("release_scratch", &release_device_scratch,
            "Free the device scratch the context-free level-1 API keeps between calls");
    mod.def("kernel_launch_count", &acg_kernel_launch_count,
            "Device kernels launched by this process through libacg_cuda.so");
}
