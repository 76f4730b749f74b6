#pragma once
// Drop-in for proj/include/anisocg/operator.hpp. OperatorContext<T> keeps the
// reference's host-side accessors and additionally owns the device context
// (profile + per-column geometry in HBM, slab placement). apply / precondition
// and the two fused sweeps run as sm_100a kernels (acg.h); host fields are
// uploaded and downloaded at the call edges, as the reference's API requires.
#include <memory>
#include <stdexcept>
#include <utility>
#include <vector>

#include "acg.h"
#include "anisocg/field.hpp"
#include "anisocg/grid.hpp"
#include "anisocg/profile.hpp"

namespace anisocg {

namespace detail {
std::shared_ptr<acg_context> make_device_context(acg_dtype dtype, const VerticalProfile& profile,
                                                 const PanelGeometry& geometry,
                                                 const acg_placement* placement);
}  // namespace detail

/// operator.hpp:29-67
template <typename T>
class OperatorContext {
public:
    OperatorContext(const VerticalProfile& profile, const PanelGeometry& geometry,
                    const acg_placement* placement = nullptr)
        : m_(geometry.m), n_z_(profile.n_z) {
        if (m_ < 1 || n_z_ < 1)
            throw std::invalid_argument("OperatorContext: empty profile or geometry");
        a_prime_.assign(profile.a_prime.begin(), profile.a_prime.end());
        b_prime_.assign(profile.b_prime.begin(), profile.b_prime.end());
        c_prime_.assign(profile.c_prime.begin(), profile.c_prime.end());
        d_.assign(profile.d.begin(), profile.d.end());
        cell_area_.assign(geometry.cell_area.begin(), geometry.cell_area.end());
        alpha_east_.assign(geometry.alpha_east.begin(), geometry.alpha_east.end());
        alpha_north_.assign(geometry.alpha_north.begin(), geometry.alpha_north.end());
        alpha_diag_.assign(geometry.alpha_diag.begin(), geometry.alpha_diag.end());
        dev_ = detail::make_device_context(detail::dtype_of<T>(), profile, geometry, placement);
    }

    int m() const { return m_; }
    int n_z() const { return n_z_; }
    std::size_t n() const { return static_cast<std::size_t>(m_) * m_ * n_z_; }
    const T* a_prime() const { return a_prime_.data(); }
    const T* b_prime() const { return b_prime_.data(); }
    const T* c_prime() const { return c_prime_.data(); }
    const T* d() const { return d_.data(); }
    T area(int i, int j) const { return cell_area_[static_cast<std::size_t>(i) * m_ + j]; }
    T alpha_diag(int i, int j) const { return alpha_diag_[static_cast<std::size_t>(i) * m_ + j]; }
    T alpha_east(int i, int j) const { return alpha_east_[static_cast<std::size_t>(i) * m_ + j]; }
    T alpha_north(int i, int j) const {
        return alpha_north_[static_cast<std::size_t>(i) * (m_ - 1) + j];
    }
    /// The device context (C ABI handle).
    acg_context* device() const { return dev_.get(); }

private:
    int m_, n_z_;
    std::vector<T> a_prime_, b_prime_, c_prime_, d_;
    std::vector<T> cell_area_, alpha_east_, alpha_north_, alpha_diag_;
    std::shared_ptr<acg_context> dev_;
};

namespace detail {
template <typename T>
void check_operand(const OperatorContext<T>& ctx, const Field3D<T>& a, const Field3D<T>& b,
                   const char* what) {
    require_conformant(a, b, what);
    if (a.m() != ctx.m() || a.n_z() != ctx.n_z())
        throw std::invalid_argument(std::string(what) + ": field does not match operator context");
}
}  // namespace detail

/// operator.hpp:101-135  y <- A x
template <typename T>
void apply(const OperatorContext<T>& ctx, const Field3D<T>& x, Field3D<T>& y, int workers = 1) {
    (void)workers;
    detail::check_operand(ctx, x, y, "apply");
    if (x.data() == y.data()) throw std::invalid_argument("apply: x and y must not alias");
    detail::check(acg_apply_host(ctx.device(), detail::layout_of(x.layout()), x.data(), y.data()));
}

/// operator.hpp:141-191  x <- M^-1 y (per-column Thomas)
template <typename T>
void precondition(const OperatorContext<T>& ctx, const Field3D<T>& y, Field3D<T>& x,
                  int workers = 1) {
    (void)workers;
    detail::check_operand(ctx, y, x, "precondition");
    if (y.data() == x.data()) throw std::invalid_argument("precondition: y and x must not alias");
    detail::check(
        acg_precondition_host(ctx.device(), detail::layout_of(y.layout()), y.data(), x.data()));
}

/// operator.hpp:195-208
template <typename T>
struct FusedState {
    Field3D<T> u, r, z, p, q;
    T alpha = T(0), beta = T(0), kappa = T(0), kappa_old = T(0), sigma = T(0), r_norm = T(0);
    FusedState(int m, int n_z, Layout layout)
        : u(m, n_z, layout), r(m, n_z, layout), z(m, n_z, layout), p(m, n_z, layout),
          q(m, n_z, layout) {}
};

/// operator.hpp:214-266 (paper Alg. 2)
template <typename T>
T interleaved_spmv_kernel(const OperatorContext<T>& ctx, FusedState<T>& st, int workers = 1) {
    (void)workers;
    require_conformant(st.u, st.z, "interleaved_spmv_kernel");
    if (st.u.m() != ctx.m() || st.u.n_z() != ctx.n_z())
        throw std::invalid_argument("interleaved_spmv_kernel: state does not match context");
    detail::Scratch u(ctx.device()), p(ctx.device()), q(ctx.device()), z(ctx.device());
    detail::upload(u.f, st.u);
    detail::upload(p.f, st.p);
    detail::upload(q.f, st.q);
    detail::upload(z.f, st.z);
    double sigma = 0;
    detail::check(acg_interleaved_spmv_kernel(ctx.device(), u.f, p.f, q.f, z.f,
                                              static_cast<double>(st.alpha),
                                              static_cast<double>(st.beta), &sigma));
    detail::download(u.f, st.u);
    detail::download(p.f, st.p);
    detail::download(q.f, st.q);
    st.sigma = static_cast<T>(sigma);
    return st.sigma;
}

/// operator.hpp:272-346 (paper Alg. 3)
template <typename T>
std::pair<T, T> interleaved_prec_kernel(const OperatorContext<T>& ctx, FusedState<T>& st,
                                        int workers = 1) {
    (void)workers;
    require_conformant(st.r, st.z, "interleaved_prec_kernel");
    if (st.r.m() != ctx.m() || st.r.n_z() != ctx.n_z())
        throw std::invalid_argument("interleaved_prec_kernel: state does not match context");
    detail::Scratch r(ctx.device()), z(ctx.device()), q(ctx.device());
    detail::upload(r.f, st.r);
    detail::upload(q.f, st.q);
    double rn = 0, ka = 0;
    detail::check(acg_interleaved_prec_kernel(ctx.device(), r.f, z.f, q.f,
                                              static_cast<double>(st.alpha), &rn, &ka));
    detail::download(r.f, st.r);
    detail::download(z.f, st.z);
    st.r_norm = static_cast<T>(rn);
    st.kappa = static_cast<T>(ka);
    return {st.r_norm, st.kappa};
}

}  // namespace anisocg
