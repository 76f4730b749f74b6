#pragma once
// Drop-in for the reference's anisocg/field.hpp (proj/include/anisocg/field.hpp):
// same Layout / linear_index / LayoutStrides / Field3D<T> API and the same
// level-1 operations, but every arithmetic operation runs in the sm_100a
// kernels behind the C ABI (include/acg.h). Field3D<T> stays host memory owned
// by the caller, exactly as in the reference (field.hpp:57-93).
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "acg.h"

namespace anisocg {

/// Thrown on a zero pivot or a CG scalar losing positivity (operator.hpp:21-24).
class NumericalBreakdown : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

/// field.hpp:21
enum class Layout { VerticalContiguous, HorizontalContiguous };

/// field.hpp:23-28
inline std::size_t linear_index(Layout layout, int i, int j, int k, int m, int n_z) {
    assert(i >= 0 && i < m && j >= 0 && j < m && k >= 0 && k < n_z);
    return layout == Layout::VerticalContiguous
               ? static_cast<std::size_t>(n_z) * (static_cast<std::size_t>(m) * i + j) + k
               : static_cast<std::size_t>(m) * (static_cast<std::size_t>(n_z) * j + k) + i;
}

/// field.hpp:34-52
struct LayoutStrides {
    std::ptrdiff_t k_stride, east, north;
    LayoutStrides(Layout layout, int m, int n_z)
        : k_stride(layout == Layout::VerticalContiguous ? 1 : m),
          east(layout == Layout::VerticalContiguous ? static_cast<std::ptrdiff_t>(n_z) * m : 1),
          north(layout == Layout::VerticalContiguous ? n_z : static_cast<std::ptrdiff_t>(m) * n_z) {}
    std::size_t column_base(Layout layout, int i, int j, int m, int n_z) const {
        return linear_index(layout, i, j, 0, m, n_z);
    }
};

template <typename T>
class Field3D {
public:
    Field3D() = default;
    Field3D(int m, int n_z, Layout layout, T fill = T(0)) : m_(m), n_z_(n_z), layout_(layout) {
        if (m < 1 || n_z < 1) throw std::invalid_argument("Field3D: m and n_z must be >= 1");
        data_.assign(static_cast<std::size_t>(m) * m * n_z, fill);
    }
    int m() const { return m_; }
    int n_z() const { return n_z_; }
    Layout layout() const { return layout_; }
    std::size_t size() const { return data_.size(); }
    std::size_t columns() const { return static_cast<std::size_t>(m_) * m_; }
    T* data() { return data_.data(); }
    const T* data() const { return data_.data(); }
    T& operator()(int i, int j, int k) { return data_[linear_index(layout_, i, j, k, m_, n_z_)]; }
    const T& operator()(int i, int j, int k) const {
        return data_[linear_index(layout_, i, j, k, m_, n_z_)];
    }
    T& operator[](std::size_t l) { return data_[l]; }
    const T& operator[](std::size_t l) const { return data_[l]; }
    bool conforms(const Field3D& o) const {
        return m_ == o.m_ && n_z_ == o.n_z_ && layout_ == o.layout_;
    }

private:
    int m_ = 0, n_z_ = 0;
    Layout layout_ = Layout::VerticalContiguous;
    std::vector<T> data_;
};

template <typename T>
inline void require_conformant(const Field3D<T>& a, const Field3D<T>& b, const char* what) {
    if (!a.conforms(b)) throw std::invalid_argument(std::string(what) + ": shape/layout mismatch");
}

namespace detail {

/// acg_status -> the reference's exception types.
void check(acg_status st);

template <typename T>
constexpr acg_dtype dtype_of() {
    return sizeof(T) == 4 ? ACG_F32 : ACG_F64;
}
inline acg_layout layout_of(Layout l) {
    return l == Layout::VerticalContiguous ? ACG_LAYOUT_VERTICAL : ACG_LAYOUT_HORIZONTAL;
}

/// Device context for context-free field operations (zero operator; shape only).
acg_context* shape_context(acg_dtype dtype, int m, int n_z);
/// Frees a context's pooled scratch fields, cached solver state and staging.
void release_scratch(const acg_context* c);

/// Scratch device field of a context, returned to a per-context pool on release.
struct Scratch {
    acg_context* ctx;
    acg_field* f;
    explicit Scratch(const acg_context* c);
    ~Scratch();
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
};

template <typename T>
void upload(acg_field* f, const Field3D<T>& x) {
    check(acg_field_upload(f, x.data(), layout_of(x.layout()), ACG_HOST_FULL));
}
template <typename T>
void download(const acg_field* f, Field3D<T>& x) {
    check(acg_field_download(f, x.data(), layout_of(x.layout()), ACG_HOST_FULL));
}

}  // namespace detail

/// Frees the device scratch the host API keeps between calls (pooled
/// fields, staging buffers, cached solver state of the shape-only contexts);
/// it is re-created on demand.
void release_device_scratch();

/// field.hpp:102-109 — value-preserving permutation (pure data movement).
template <typename T>
Field3D<T> relayout(const Field3D<T>& x, Layout target) {
    Field3D<T> out(x.m(), x.n_z(), target);
    for (int i = 0; i < x.m(); ++i)
        for (int j = 0; j < x.m(); ++j)
            for (int k = 0; k < x.n_z(); ++k) out(i, j, k) = x(i, j, k);
    return out;
}

/// field.hpp:116-124  y <- alpha x + y (GPU)
template <typename T>
void axpy(T alpha, const Field3D<T>& x, Field3D<T>& y, int workers = 1) {
    (void)workers;
    require_conformant(x, y, "axpy");
    acg_context* c = detail::shape_context(detail::dtype_of<T>(), x.m(), x.n_z());
    detail::Scratch fx(c), fy(c);
    detail::upload(fx.f, x);
    detail::upload(fy.f, y);
    detail::check(acg_axpy(static_cast<double>(alpha), fx.f, fy.f));
    detail::download(fy.f, y);
}

/// field.hpp:126-132  x <- alpha x (GPU)
template <typename T>
void scal(T alpha, Field3D<T>& x, int workers = 1) {
    (void)workers;
    acg_context* c = detail::shape_context(detail::dtype_of<T>(), x.m(), x.n_z());
    detail::Scratch fx(c);
    detail::upload(fx.f, x);
    detail::check(acg_scal(static_cast<double>(alpha), fx.f));
    detail::download(fx.f, x);
}

/// field.hpp:134-153 — per-column sums in ascending k, pairwise over columns (GPU)
template <typename T>
T dot(const Field3D<T>& x, const Field3D<T>& y, int workers = 1) {
    (void)workers;
    require_conformant(x, y, "dot");
    acg_context* c = detail::shape_context(detail::dtype_of<T>(), x.m(), x.n_z());
    detail::Scratch fx(c), fy(c);
    detail::upload(fx.f, x);
    detail::upload(fy.f, y);
    double out = 0;
    detail::check(acg_dot(fx.f, fy.f, &out));
    return static_cast<T>(out);
}

/// field.hpp:155-173 (GPU)
template <typename T>
T nrm2(const Field3D<T>& x, int workers = 1) {
    (void)workers;
    acg_context* c = detail::shape_context(detail::dtype_of<T>(), x.m(), x.n_z());
    detail::Scratch fx(c);
    detail::upload(fx.f, x);
    double out = 0;
    detail::check(acg_nrm2(fx.f, &out));
    return static_cast<T>(out);
}

/// field.hpp:180-196 — splitmix64 in canonical (i,j,k) order, generated on the GPU
template <typename T>
void fill_random(Field3D<T>& x, std::uint64_t seed) {
    acg_context* c = detail::shape_context(detail::dtype_of<T>(), x.m(), x.n_z());
    detail::Scratch fx(c);
    detail::check(acg_field_fill_random(fx.f, seed));
    detail::download(fx.f, x);
}

}  // namespace anisocg
