// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// C-ABI harness around the UNMODIFIED reference hot path, compiled from the
// sources where they lie under /root/reference/proj (headers + src/grid.cpp +
// src/profile.cpp) by oracle/Makefile into oracle/_ref/libanisocg_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// --impl reference) load it, as the checker / the CPU baseline.
//
// Every entry point forwards to the reference template of the same name:
//   apply                  proj/include/anisocg/operator.hpp:101-135
//   precondition           proj/include/anisocg/operator.hpp:141-191
//   interleaved_spmv_kernel proj/include/anisocg/operator.hpp:214-266
//   interleaved_prec_kernel proj/include/anisocg/operator.hpp:272-346
//   solve / pcg_*          proj/include/anisocg/solver.hpp:162-378
//   true_residual          proj/include/anisocg/solver.hpp:61-69
//   fill_random, dot, nrm2 proj/include/anisocg/field.hpp:134-196
// Status codes: 0 ok, 1 std::invalid_argument, 2 NumericalBreakdown, 5 other.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>

#include "anisocg/field.hpp"
#include "anisocg/grid.hpp"
#include "anisocg/operator.hpp"
#include "anisocg/profile.hpp"
#include "anisocg/solver.hpp"

using namespace anisocg;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const NumericalBreakdown& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

struct RefCtx {
    PanelGeometry geometry;
    VerticalGrid vgrid;
    VerticalProfile profile;
    std::unique_ptr<OperatorContext<double>> c64;
    std::unique_ptr<OperatorContext<float>> c32;
};

Layout lay(int layout) {
    return layout == 1 ? Layout::HorizontalContiguous : Layout::VerticalContiguous;
}

template <typename T>
Field3D<T> in_field(const RefCtx& c, int layout, const void* data) {
    Field3D<T> f(c.geometry.m, c.vgrid.n_z, lay(layout));
    std::memcpy(f.data(), data, f.size() * sizeof(T));
    return f;
}

template <typename T>
void out_field(const Field3D<T>& f, void* data) {
    std::memcpy(data, f.data(), f.size() * sizeof(T));
}

template <typename T>
const OperatorContext<T>& ctx_of(const RefCtx& c);
template <>
const OperatorContext<double>& ctx_of<double>(const RefCtx& c) { return *c.c64; }
template <>
const OperatorContext<float>& ctx_of<float>(const RefCtx& c) { return *c.c32; }

}  // namespace

extern "C" {

struct ref_result {
    int iterations;
    int converged;
    double true_residual;
    int n_residual, n_kappa, n_alpha, n_beta;
    double fused_prec_s, fused_spmv_s, spmv_s, prec_s, blas_s, setup_s, total_s;
};

const char* ref_last_error() { return g_err.c_str(); }

int ref_vertical_grid(int n_z, double h, double* r_out) {
    return guard([&] {
        const auto g = build_graded_vertical_grid(n_z, h);
        std::memcpy(r_out, g.r.data(), g.r.size() * sizeof(double));
    });
}

// kind 0 = cubed sphere, 1 = planar. Arrays: area m*m, east (m-1)*m, north m*(m-1), diag m*m.
int ref_panel(int kind, int m, double extent, double* area, double* east, double* north,
              double* diag) {
    return guard([&] {
        const auto g = kind == 0 ? build_cubed_sphere_panel(m) : build_planar_panel(m, extent);
        std::memcpy(area, g.cell_area.data(), g.cell_area.size() * sizeof(double));
        std::memcpy(east, g.alpha_east.data(), g.alpha_east.size() * sizeof(double));
        std::memcpy(north, g.alpha_north.data(), g.alpha_north.size() * sizeof(double));
        std::memcpy(diag, g.alpha_diag.data(), g.alpha_diag.size() * sizeof(double));
    });
}

int ref_profile(int n_z, double h, double omega2, double lambda2, double* ap, double* bp,
                double* cp, double* d) {
    return guard([&] {
        const auto p = build_vertical_profile(build_graded_vertical_grid(n_z, h), omega2, lambda2);
        std::memcpy(ap, p.a_prime.data(), n_z * sizeof(double));
        std::memcpy(bp, p.b_prime.data(), n_z * sizeof(double));
        std::memcpy(cp, p.c_prime.data(), n_z * sizeof(double));
        std::memcpy(d, p.d.data(), n_z * sizeof(double));
    });
}

int ref_anisotropy(int kind, int m, double extent, int n_z, double h, double lambda2,
                   double* out) {
    return guard([&] {
        const auto g = kind == 0 ? build_cubed_sphere_panel(m) : build_planar_panel(m, extent);
        const auto a = anisotropy(g, build_graded_vertical_grid(n_z, h), lambda2);
        std::memcpy(out, a.data(), a.size() * sizeof(double));
    });
}

// Builds geometry + grid + profile like the reference fixtures
// (tests/test_operator.cpp:12-28) and both precision contexts.
// flip_d != 0 negates d (the non-SPD fixture of tests/test_solver.cpp:194-204).
void* ref_ctx_create(int kind, int m, int n_z, double h, double extent, double omega2,
                     double lambda2, int flip_d) {
    RefCtx* c = nullptr;
    const int st = guard([&] {
        auto p = std::make_unique<RefCtx>();
        p->geometry = kind == 0 ? build_cubed_sphere_panel(m) : build_planar_panel(m, extent);
        p->vgrid = build_graded_vertical_grid(n_z, h);
        p->profile = build_vertical_profile(p->vgrid, omega2, lambda2);
        if (flip_d)
            for (auto& v : p->profile.d) v = -v;
        p->c64 = std::make_unique<OperatorContext<double>>(p->profile, p->geometry);
        p->c32 = std::make_unique<OperatorContext<float>>(p->profile, p->geometry);
        c = p.release();
    });
    return st == 0 ? c : nullptr;
}

void ref_ctx_destroy(void* c) { delete static_cast<RefCtx*>(c); }

#define REF_DISPATCH(dtype, ...)              \
    do {                                       \
        if ((dtype) == 1) {                    \
            using T = float;                   \
            __VA_ARGS__;                       \
        } else {                               \
            using T = double;                  \
            __VA_ARGS__;                       \
        }                                      \
    } while (0)

int ref_fill_random(int dtype, int layout, int m, int n_z, std::uint64_t seed, void* out) {
    return guard([&] {
        REF_DISPATCH(dtype, {
            Field3D<T> f(m, n_z, lay(layout));
            fill_random(f, seed);
            out_field(f, out);
        });
    });
}

int ref_apply(void* cp, int dtype, int layout, const void* x, void* y, int workers) {
    const RefCtx& c = *static_cast<RefCtx*>(cp);
    return guard([&] {
        REF_DISPATCH(dtype, {
            auto xf = in_field<T>(c, layout, x);
            Field3D<T> yf(c.geometry.m, c.vgrid.n_z, lay(layout));
            apply(ctx_of<T>(c), xf, yf, workers);
            out_field(yf, y);
        });
    });
}

int ref_precondition(void* cp, int dtype, int layout, const void* y, void* x, int workers) {
    const RefCtx& c = *static_cast<RefCtx*>(cp);
    return guard([&] {
        REF_DISPATCH(dtype, {
            auto yf = in_field<T>(c, layout, y);
            Field3D<T> xf(c.geometry.m, c.vgrid.n_z, lay(layout));
            precondition(ctx_of<T>(c), yf, xf, workers);
            out_field(xf, x);
        });
    });
}

// In/out fields u, p, q; in z. sigma returned as double.
int ref_fused_spmv(void* cp, int dtype, int layout, void* u, void* p, void* q, const void* z,
                   double alpha, double beta, double* sigma, int workers) {
    const RefCtx& c = *static_cast<RefCtx*>(cp);
    return guard([&] {
        REF_DISPATCH(dtype, {
            FusedState<T> st(c.geometry.m, c.vgrid.n_z, lay(layout));
            st.u = in_field<T>(c, layout, u);
            st.p = in_field<T>(c, layout, p);
            st.q = in_field<T>(c, layout, q);
            st.z = in_field<T>(c, layout, z);
            st.alpha = static_cast<T>(alpha);
            st.beta = static_cast<T>(beta);
            *sigma = static_cast<double>(interleaved_spmv_kernel(ctx_of<T>(c), st, workers));
            out_field(st.u, u);
            out_field(st.p, p);
            out_field(st.q, q);
        });
    });
}

// In/out r, out z, in q.
int ref_fused_prec(void* cp, int dtype, int layout, void* r, void* z, const void* q,
                   double alpha, double* r_norm, double* kappa, int workers) {
    const RefCtx& c = *static_cast<RefCtx*>(cp);
    return guard([&] {
        REF_DISPATCH(dtype, {
            FusedState<T> st(c.geometry.m, c.vgrid.n_z, lay(layout));
            st.r = in_field<T>(c, layout, r);
            st.q = in_field<T>(c, layout, q);
            st.alpha = static_cast<T>(alpha);
            const auto pr = interleaved_prec_kernel(ctx_of<T>(c), st, workers);
            *r_norm = static_cast<double>(pr.first);
            *kappa = static_cast<double>(pr.second);
            out_field(st.r, r);
            out_field(st.z, z);
        });
    });
}

int ref_dot(void* cp, int dtype, int layout, const void* x, const void* y, double* out,
            int workers) {
    const RefCtx& c = *static_cast<RefCtx*>(cp);
    return guard([&] {
        REF_DISPATCH(dtype, {
            *out = static_cast<double>(
                dot(in_field<T>(c, layout, x), in_field<T>(c, layout, y), workers));
        });
    });
}

int ref_nrm2(void* cp, int dtype, int layout, const void* x, double* out, int workers) {
    const RefCtx& c = *static_cast<RefCtx*>(cp);
    return guard([&] {
        REF_DISPATCH(dtype,
                     { *out = static_cast<double>(nrm2(in_field<T>(c, layout, x), workers)); });
    });
}

int ref_true_residual(void* cp, int dtype, int layout, const void* u, const void* f,
                      double* out, int workers) {
    const RefCtx& c = *static_cast<RefCtx*>(cp);
    return guard([&] {
        REF_DISPATCH(dtype, {
            *out = static_cast<double>(true_residual(
                ctx_of<T>(c), in_field<T>(c, layout, u), in_field<T>(c, layout, f), workers));
        });
    });
}

// variant: 0 standard, 1 interleaved, 2 standard on the CsrBackend
// (backend = csr, solver.hpp:126-145). Histories are written into caller
// buffers of capacity maxiter + 2; u0 may be null (zero start).
int ref_solve(void* cp, int dtype, int layout, const void* f, const void* u0, double epsilon,
              double tau, int maxiter, int variant, int workers, void* u_out, ref_result* res,
              double* residual_h, double* kappa_h, double* alpha_h, double* beta_h) {
    const RefCtx& c = *static_cast<RefCtx*>(cp);
    return guard([&] {
        REF_DISPATCH(dtype, {
            SolverConfig cfg;
            cfg.epsilon = epsilon;
            cfg.tau = tau;
            cfg.maxiter = maxiter;
            cfg.workers = workers;
            cfg.variant = variant == 1 ? Variant::interleaved : Variant::standard;
            cfg.backend = variant == 2 ? BackendKind::csr : BackendKind::matrix_free;
            auto ff = in_field<T>(c, layout, f);
            Field3D<T> uu(c.geometry.m, c.vgrid.n_z, lay(layout));
            if (u0) uu = in_field<T>(c, layout, u0);
            auto [u, r] = solve(ctx_of<T>(c), ff, uu, cfg);
            out_field(u, u_out);
            res->iterations = r.iterations;
            res->converged = r.converged ? 1 : 0;
            res->true_residual = r.true_residual;
            res->n_residual = static_cast<int>(r.residual_history.size());
            res->n_kappa = static_cast<int>(r.kappa_history.size());
            res->n_alpha = static_cast<int>(r.alpha_history.size());
            res->n_beta = static_cast<int>(r.beta_history.size());
            res->fused_prec_s = r.timings.fused_prec;
            res->fused_spmv_s = r.timings.fused_spmv;
            res->spmv_s = r.timings.spmv;
            res->prec_s = r.timings.prec;
            res->blas_s = r.timings.blas;
            res->setup_s = r.timings.setup;
            res->total_s = r.timings.total;
            std::memcpy(residual_h, r.residual_history.data(),
                        r.residual_history.size() * sizeof(double));
            std::memcpy(kappa_h, r.kappa_history.data(), r.kappa_history.size() * sizeof(double));
            std::memcpy(alpha_h, r.alpha_history.data(), r.alpha_history.size() * sizeof(double));
            std::memcpy(beta_h, r.beta_history.data(), r.beta_history.size() * sizeof(double));
        });
    });
}

}  // extern "C"
