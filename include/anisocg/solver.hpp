#pragma once
// Drop-in for proj/include/anisocg/solver.hpp. The PCG drivers run device
// resident (acg_solve_host): the scalar recurrences of solver.hpp:288-364 are
// evaluated on the GPU between the sweeps, so the loop has no host sync per
// iteration. Histories, counts and exit semantics match the reference.
#include <stdexcept>
#include <utility>
#include <vector>

#include "acg.h"
#include "anisocg/csr.hpp"
#include "anisocg/field.hpp"
#include "anisocg/operator.hpp"

namespace anisocg {

enum class Variant { standard, interleaved };
enum class BackendKind { matrix_free, csr };

/// solver.hpp:19-36
struct SolverConfig {
    double epsilon = 1e-5;
    double tau = 1e-20;
    int maxiter = 500;
    Variant variant = Variant::standard;
    BackendKind backend = BackendKind::matrix_free;
    int workers = 1;

    void validate() const {
        if (!(epsilon > 0.0)) throw std::invalid_argument("SolverConfig: epsilon must be > 0");
        if (!(tau > 0.0)) throw std::invalid_argument("SolverConfig: tau must be > 0");
        if (maxiter < 1) throw std::invalid_argument("SolverConfig: maxiter must be >= 1");
        if (workers < 1) throw std::invalid_argument("SolverConfig: workers must be >= 1");
        if (variant == Variant::interleaved && backend == BackendKind::csr)
            throw std::invalid_argument(
                "SolverConfig: the interleaved variant exists for the matrix-free backend only");
    }
};

/// solver.hpp:39-47 (seconds; device times from CUDA events)
struct KernelTimings {
    double spmv = 0.0, prec = 0.0, blas = 0.0, fused_spmv = 0.0, fused_prec = 0.0;
    double setup = 0.0, total = 0.0;
};

/// solver.hpp:49-58
struct SolveResult {
    int iterations = 0;
    bool converged = false;
    std::vector<double> residual_history;
    std::vector<double> kappa_history;
    std::vector<double> alpha_history;
    std::vector<double> beta_history;
    double true_residual = 0.0;
    KernelTimings timings;
};

/// solver.hpp:61-69 — ||f - A u|| (one fused device pass)
template <typename T>
T true_residual(const OperatorContext<T>& ctx, const Field3D<T>& u, const Field3D<T>& f,
                int workers = 1) {
    (void)workers;
    detail::check_operand(ctx, u, f, "true_residual");
    double out = 0;
    detail::check(acg_true_residual_host(ctx.device(), detail::layout_of(u.layout()), u.data(),
                                         f.data(), &out));
    return static_cast<T>(out);
}

/// solver.hpp:71-78 — ||f - A u|| with a stored matrix (host spmv_csr, then
/// the device level-1 operations of field.hpp)
template <typename T>
T true_residual(const CsrMatrix<T>& A, const Field3D<T>& u, const Field3D<T>& f, int workers = 1) {
    Field3D<T> t(u.m(), u.n_z(), u.layout());
    spmv_csr(A, u, t, workers);
    scal(T(-1), t, workers);
    axpy(T(1), f, t, workers);
    return nrm2(t, workers);
}

namespace detail {
template <typename T>
std::pair<Field3D<T>, SolveResult> run_solve(const OperatorContext<T>& ctx, const Field3D<T>& f,
                                             const Field3D<T>& u0, const SolverConfig& cfg,
                                             Variant variant, const char* what) {
    cfg.validate();
    require_conformant(f, u0, what);
    if (f.m() != ctx.m() || f.n_z() != ctx.n_z())
        throw std::invalid_argument(std::string(what) + ": fields do not match operator context");
    acg_solver_config c{};
    acg_solver_config_default(&c);
    c.epsilon = cfg.epsilon;
    c.tau = cfg.tau;
    c.maxiter = cfg.maxiter;
    c.workers = cfg.workers;
    c.variant = variant == Variant::interleaved ? ACG_VARIANT_INTERLEAVED : ACG_VARIANT_STANDARD;
    // CsrBackend (solver.hpp:126-145): stored CSR + tridiagonals on the GPU
    c.backend = cfg.backend == BackendKind::csr ? ACG_BACKEND_CSR : ACG_BACKEND_MATRIX_FREE;
    c.layout = layout_of(f.layout());
    c.record_timings = 1;
    Field3D<T> u(f.m(), f.n_z(), f.layout());
    acg_solve_result r{};
    // NULL history buffers: the library returns exactly the pushed entries
    // (no maxiter-sized allocation, like the reference's push_back histories)
    check(acg_solve_host(ctx.device(), layout_of(f.layout()), f.data(), u0.data(), &c, u.data(),
                         &r, nullptr, nullptr, nullptr, nullptr));
    SolveResult res;
    res.iterations = r.iterations;
    res.converged = r.converged != 0;
    res.true_residual = r.true_residual;
    res.residual_history.assign(r.history[0], r.history[0] + r.n_residual);
    res.kappa_history.assign(r.history[1], r.history[1] + r.n_kappa);
    res.alpha_history.assign(r.history[2], r.history[2] + r.n_alpha);
    res.beta_history.assign(r.history[3], r.history[3] + r.n_beta);
    acg_solve_result_release(&r);
    res.timings.spmv = r.timings.spmv;
    res.timings.prec = r.timings.prec;
    res.timings.blas = r.timings.blas;
    res.timings.fused_spmv = r.timings.fused_spmv;
    res.timings.fused_prec = r.timings.fused_prec;
    res.timings.setup = r.timings.setup;
    res.timings.total = r.timings.total;
    return {std::move(u), std::move(res)};
}
}  // namespace detail

/// solver.hpp:162-268
template <typename T>
std::pair<Field3D<T>, SolveResult> pcg_standard(const OperatorContext<T>& ctx, const Field3D<T>& f,
                                                const Field3D<T>& u0, const SolverConfig& cfg) {
    return detail::run_solve(ctx, f, u0, cfg, Variant::standard, "pcg_standard");
}

/// solver.hpp:275-370
template <typename T>
std::pair<Field3D<T>, SolveResult> pcg_interleaved(const OperatorContext<T>& ctx,
                                                   const Field3D<T>& f, const Field3D<T>& u0,
                                                   const SolverConfig& cfg) {
    return detail::run_solve(ctx, f, u0, cfg, Variant::interleaved, "pcg_interleaved");
}

/// solver.hpp:373-378
template <typename T>
std::pair<Field3D<T>, SolveResult> solve(const OperatorContext<T>& ctx, const Field3D<T>& f,
                                         const Field3D<T>& u0, const SolverConfig& cfg) {
    if (cfg.variant == Variant::interleaved) return pcg_interleaved(ctx, f, u0, cfg);
    return pcg_standard(ctx, f, u0, cfg);
}

}  // namespace anisocg
