"""TEST INFRASTRUCTURE ONLY — the CPU oracle (checker), never the product.

ctypes front-ends for
  * ``liboracle.so``            — the plain-C restatement (oracle/acg_oracle.c), and
  * ``_ref/libanisocg_ref.so``  — the unmodified reference hot path compiled from
                                  /root/reference (oracle/ref_harness.cpp).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg,
``--impl reference``) may import this module. The product package
``paper_1302_7193_b200`` never imports it; it fails loudly without its CUDA
library instead of falling back here.

Field arrays use the reference's own linear layouts (field.hpp:23-28):
layout 0 = VerticalContiguous (numpy shape (m, m, n_z), C order — the Python
binding convention, bindings.cpp:1-3), layout 1 = HorizontalContiguous
(numpy shape (m, n_z, m) indexed [j, k, i]).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libanisocg_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


@dataclass
class Problem:
    """Reference fixture parameters (tests/test_operator.cpp:12-28)."""

    m: int
    n_z: int
    sphere: bool = True
    omega2: float = 6.71e-4
    lambda2: float = 3.32e-2
    h: float = 1e-2
    extent: float = 2.0


@dataclass
class Result:
    iterations: int
    converged: bool
    true_residual: float
    residual_history: np.ndarray
    kappa_history: np.ndarray
    alpha_history: np.ndarray
    beta_history: np.ndarray
    status: int = 0
    timings: dict = field(default_factory=dict)


def shape_of(m, n_z, layout):
    return (m, m, n_z) if layout == 0 else (m, n_z, m)


# --------------------------------------------------------------------------
# plain-C restatement
# --------------------------------------------------------------------------
class _OrcResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("status", C.c_int),
                ("true_residual", C.c_double), ("n_residual", C.c_int), ("n_kappa", C.c_int),
                ("n_alpha", C.c_int), ("n_beta", C.c_int)]


_orc = None


def lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle not built: {ORACLE_SO} (run make -C oracle)")
        L = C.CDLL(ORACLE_SO)
        L.orc_ctx_create.restype = C.c_void_p
        L.orc_ctx_create.argtypes = [C.c_int, C.c_int] + [_dp] * 8
        L.orc_ctx_destroy.argtypes = [C.c_void_p]
        for s, ct in (("f64", C.c_double), ("f32", C.c_float)):
            getattr(L, f"orc_pairwise_sum_{s}").restype = ct
            getattr(L, f"orc_pairwise_sum_{s}").argtypes = [_vp, C.c_size_t]
            getattr(L, f"orc_fill_random_{s}").argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_uint64]
            getattr(L, f"orc_apply_{s}").argtypes = [C.c_void_p, C.c_int, _vp, _vp]
            getattr(L, f"orc_precondition_{s}").argtypes = [C.c_void_p, C.c_int, _vp, _vp]
            getattr(L, f"orc_fused_spmv_{s}").argtypes = [C.c_void_p, C.c_int, _vp, _vp, _vp, _vp,
                                                         ct, ct, C.POINTER(ct), _vp]
            getattr(L, f"orc_fused_prec_{s}").argtypes = [C.c_void_p, C.c_int, _vp, _vp, _vp, ct,
                                                         C.POINTER(ct), C.POINTER(ct), _vp, _vp]
            getattr(L, f"orc_dot_{s}").restype = ct
            getattr(L, f"orc_dot_{s}").argtypes = [C.c_int, C.c_int, C.c_int, _vp, _vp]
            getattr(L, f"orc_nrm2_{s}").restype = ct
            getattr(L, f"orc_nrm2_{s}").argtypes = [C.c_int, C.c_int, C.c_int, _vp]
            getattr(L, f"orc_true_residual_{s}").restype = ct
            getattr(L, f"orc_true_residual_{s}").argtypes = [C.c_void_p, C.c_int, _vp, _vp]
            getattr(L, f"orc_solve_{s}").argtypes = [C.c_void_p, C.c_int, _vp, _vp, C.c_double,
                                                    C.c_double, C.c_int, C.c_int, _vp,
                                                    C.POINTER(_OrcResult), _dp, _dp, _dp, _dp]
        L.orc_vertical_grid.argtypes = [C.c_int, C.c_double, _dp]
        L.orc_cubed_sphere_panel.argtypes = [C.c_int, _dp, _dp, _dp, _dp]
        L.orc_planar_panel.argtypes = [C.c_int, C.c_double, _dp, _dp, _dp, _dp]
        L.orc_vertical_profile.argtypes = [C.c_int, _dp, C.c_double, C.c_double, _dp, _dp, _dp, _dp]
        L.orc_anisotropy.argtypes = [C.c_int, _dp, C.c_int, _dp, C.c_double, _dp]
        _orc = L
    return _orc


def vertical_grid(n_z, h):
    r = np.empty(n_z + 1)
    if lib().orc_vertical_grid(n_z, h, r):
        raise ValueError("vertical_grid: bad arguments")
    return r


def panel(m, sphere=True, extent=2.0):
    """(area[m,m], east[m-1,m], north[m,m-1], diag[m,m]) — grid.hpp:30-44 indexing."""
    area, diag = np.empty((m, m)), np.empty((m, m))
    east, north = np.empty((max(m - 1, 0), m)), np.empty((m, max(m - 1, 0)))
    e1, n1 = (east if east.size else np.empty(1)), (north if north.size else np.empty(1))
    st = (lib().orc_cubed_sphere_panel(m, area, e1, n1, diag) if sphere
          else lib().orc_planar_panel(m, extent, area, e1, n1, diag))
    if st:
        raise ValueError("panel: bad arguments")
    return area, east, north, diag


def vertical_profile(r, omega2, lambda2):
    n_z = len(r) - 1
    out = [np.empty(n_z) for _ in range(4)]
    if lib().orc_vertical_profile(n_z, np.ascontiguousarray(r, dtype=np.float64), omega2, lambda2, *out):
        raise ValueError("vertical_profile: bad arguments")
    return tuple(out)  # a', b', c', d


def anisotropy(area, r, lambda2):
    m, n_z = area.shape[0], len(r) - 1
    out = np.empty((m, m, n_z))
    lib().orc_anisotropy(m, np.ascontiguousarray(area), n_z, np.ascontiguousarray(r), lambda2, out)
    return out


def _np_t(dtype):
    return np.float32 if dtype in (np.float32, "f32", 1) else np.float64


class Oracle:
    """Operator context of the C restatement (OperatorContext<T>, operator.hpp:29-67)."""

    def __init__(self, prob: Problem):
        self.prob = prob
        m, n_z = prob.m, prob.n_z
        self.r = vertical_grid(n_z, prob.h)
        self.area, self.east, self.north, self.diag = panel(m, prob.sphere, prob.extent)
        self.ap, self.bp, self.cp, self.d = vertical_profile(self.r, prob.omega2, prob.lambda2)
        self._build()

    def _build(self):
        m, n_z = self.prob.m, self.prob.n_z
        one = np.zeros(1)
        e = np.ascontiguousarray(self.east).reshape(-1) if self.east.size else one
        n = np.ascontiguousarray(self.north).reshape(-1) if self.north.size else one
        self._h = lib().orc_ctx_create(m, n_z, self.ap, self.bp, self.cp, self.d,
                                      np.ascontiguousarray(self.area).reshape(-1), e, n,
                                      np.ascontiguousarray(self.diag).reshape(-1))

    def flip_d(self):
        """Non-SPD fixture: negate d (tests/test_solver.cpp:194-204)."""
        lib().orc_ctx_destroy(self._h)
        self.d = -self.d
        self._build()
        return self

    def __del__(self):
        try:
            lib().orc_ctx_destroy(self._h)
        except Exception:
            pass

    # helpers -------------------------------------------------------------
    def _s(self, dt):
        return "f32" if dt == np.float32 else "f64"

    def _ct(self, dt):
        return C.c_float if dt == np.float32 else C.c_double

    def random_field(self, seed, dtype=np.float64, layout=0):
        dt = _np_t(dtype)
        x = np.empty(shape_of(self.prob.m, self.prob.n_z, layout), dtype=dt)
        getattr(lib(), f"orc_fill_random_{self._s(dt)}")(_ptr(x), layout, self.prob.m, self.prob.n_z, seed)
        return x

    def apply(self, x, layout=0):
        x = np.ascontiguousarray(x)
        y = np.empty_like(x)
        if getattr(lib(), f"orc_apply_{self._s(x.dtype)}")(self._h, layout, _ptr(x), _ptr(y)):
            raise ValueError("apply: aliasing")
        return y

    def precondition(self, y, layout=0):
        y = np.ascontiguousarray(y)
        x = np.empty_like(y)
        st = getattr(lib(), f"orc_precondition_{self._s(y.dtype)}")(self._h, layout, _ptr(y), _ptr(x))
        if st == 2:
            raise RuntimeError("precondition: zero pivot in tridiagonal elimination")
        return x

    def fused_spmv(self, u, p, q, z, alpha, beta, layout=0):
        """In place on copies; returns (u, p, q, sigma, column partials)."""
        u, p, q, z = (np.array(a, copy=True, order="C") for a in (u, p, q, z))
        ct = self._ct(u.dtype)
        sg = ct()
        part = np.empty(self.prob.m ** 2, dtype=u.dtype)
        getattr(lib(), f"orc_fused_spmv_{self._s(u.dtype)}")(
            self._h, layout, _ptr(u), _ptr(p), _ptr(q), _ptr(z), alpha, beta, C.byref(sg), _ptr(part))
        return u, p, q, sg.value, part

    def fused_prec(self, r, q, alpha, layout=0):
        """Returns (r, z, r_norm, kappa, r2 partials, kappa partials)."""
        r = np.array(r, copy=True, order="C")
        q = np.ascontiguousarray(q)
        z = np.zeros_like(r)
        ct = self._ct(r.dtype)
        rn, ka = ct(), ct()
        p2 = np.empty(self.prob.m ** 2, dtype=r.dtype)
        pk = np.empty_like(p2)
        st = getattr(lib(), f"orc_fused_prec_{self._s(r.dtype)}")(
            self._h, layout, _ptr(r), _ptr(z), _ptr(q), alpha, C.byref(rn), C.byref(ka), _ptr(p2), _ptr(pk))
        if st == 2:
            raise RuntimeError("interleaved_prec_kernel: zero pivot in tridiagonal elimination")
        return r, z, rn.value, ka.value, p2, pk

    def dot(self, x, y, layout=0):
        return getattr(lib(), f"orc_dot_{self._s(x.dtype)}")(layout, self.prob.m, self.prob.n_z,
                                                          _ptr(np.ascontiguousarray(x)), _ptr(np.ascontiguousarray(y)))

    def nrm2(self, x, layout=0):
        return getattr(lib(), f"orc_nrm2_{self._s(x.dtype)}")(layout, self.prob.m, self.prob.n_z,
                                                           _ptr(np.ascontiguousarray(x)))

    def true_residual(self, u, f, layout=0):
        return getattr(lib(), f"orc_true_residual_{self._s(u.dtype)}")(
            self._h, layout, _ptr(np.ascontiguousarray(u)), _ptr(np.ascontiguousarray(f)))

    def solve(self, f, u0=None, epsilon=1e-5, tau=1e-20, maxiter=500, variant="interleaved", layout=0):
        f = np.ascontiguousarray(f)
        u = np.empty_like(f)
        cap = maxiter + 2
        hs = [np.zeros(cap) for _ in range(4)]
        res = _OrcResult()
        st = getattr(lib(), f"orc_solve_{self._s(f.dtype)}")(
            self._h, layout, _ptr(f), _ptr(np.ascontiguousarray(u0) if u0 is not None else None),
            epsilon, tau, maxiter, 1 if variant == "interleaved" else 0, _ptr(u), C.byref(res), *hs)
        if st == 1:
            raise ValueError("solve: bad configuration")
        if st == 2:
            raise RuntimeError("numerical breakdown")
        return u, Result(res.iterations, bool(res.converged), res.true_residual,
                         hs[0][:res.n_residual].copy(), hs[1][:res.n_kappa].copy(),
                         hs[2][:res.n_alpha].copy(), hs[3][:res.n_beta].copy(), st)

    def pairwise_sum(self, v):
        v = np.ascontiguousarray(v)
        return getattr(lib(), f"orc_pairwise_sum_{self._s(v.dtype)}")(_ptr(v), v.size)


# --------------------------------------------------------------------------
# the reference itself (compiled from /root/reference into oracle/_ref)
# --------------------------------------------------------------------------
class _RefResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("true_residual", C.c_double),
                ("n_residual", C.c_int), ("n_kappa", C.c_int), ("n_alpha", C.c_int),
                ("n_beta", C.c_int), ("fused_prec_s", C.c_double), ("fused_spmv_s", C.c_double),
                ("spmv_s", C.c_double), ("prec_s", C.c_double), ("blas_s", C.c_double),
                ("setup_s", C.c_double), ("total_s", C.c_double)]


_ref = None


def ref_available():
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference not built: {REF_SO} (run make -C oracle in the container)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_vertical_grid.argtypes = [C.c_int, C.c_double, _dp]
        L.ref_panel.argtypes = [C.c_int, C.c_int, C.c_double, _vp, _vp, _vp, _vp]
        L.ref_profile.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp, _dp, _dp]
        L.ref_anisotropy.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, _dp]
        L.ref_ctx_create.restype = C.c_void_p
        L.ref_ctx_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_int]
        L.ref_ctx_destroy.argtypes = [C.c_void_p]
        L.ref_fill_random.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, _vp]
        L.ref_apply.argtypes = [C.c_void_p, C.c_int, C.c_int, _vp, _vp, C.c_int]
        L.ref_precondition.argtypes = [C.c_void_p, C.c_int, C.c_int, _vp, _vp, C.c_int]
        L.ref_fused_spmv.argtypes = [C.c_void_p, C.c_int, C.c_int, _vp, _vp, _vp, _vp, C.c_double,
                                     C.c_double, C.POINTER(C.c_double), C.c_int]
        L.ref_fused_prec.argtypes = [C.c_void_p, C.c_int, C.c_int, _vp, _vp, _vp, C.c_double,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int]
        L.ref_dot.argtypes = [C.c_void_p, C.c_int, C.c_int, _vp, _vp, C.POINTER(C.c_double), C.c_int]
        L.ref_nrm2.argtypes = [C.c_void_p, C.c_int, C.c_int, _vp, C.POINTER(C.c_double), C.c_int]
        L.ref_true_residual.argtypes = [C.c_void_p, C.c_int, C.c_int, _vp, _vp, C.POINTER(C.c_double), C.c_int]
        L.ref_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, _vp, _vp, C.c_double, C.c_double,
                                C.c_int, C.c_int, C.c_int, _vp, C.POINTER(_RefResult), _dp, _dp, _dp, _dp]
        _ref = L
    return _ref


def _check(st):
    if st == 0:
        return
    msg = ref_lib().ref_last_error().decode()
    if st == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


class Reference:
    """The reference's own code path (OpenMP `workers` threads), same API as Oracle."""

    def __init__(self, prob: Problem, flip_d=False, workers=1):
        self.prob = prob
        self.workers = workers
        self._h = ref_lib().ref_ctx_create(0 if prob.sphere else 1, prob.m, prob.n_z, prob.h,
                                          prob.extent, prob.omega2, prob.lambda2, int(flip_d))
        if not self._h:
            raise ValueError(ref_lib().ref_last_error().decode())

    def __del__(self):
        try:
            ref_lib().ref_ctx_destroy(self._h)
        except Exception:
            pass

    @staticmethod
    def _dt(a):
        return 1 if a.dtype == np.float32 else 0

    def random_field(self, seed, dtype=np.float64, layout=0):
        dt = _np_t(dtype)
        x = np.empty(shape_of(self.prob.m, self.prob.n_z, layout), dtype=dt)
        _check(ref_lib().ref_fill_random(1 if dt == np.float32 else 0, layout, self.prob.m,
                                         self.prob.n_z, seed, _ptr(x)))
        return x

    def apply(self, x, layout=0):
        x = np.ascontiguousarray(x)
        y = np.empty_like(x)
        _check(ref_lib().ref_apply(self._h, self._dt(x), layout, _ptr(x), _ptr(y), self.workers))
        return y

    def precondition(self, y, layout=0):
        y = np.ascontiguousarray(y)
        x = np.empty_like(y)
        _check(ref_lib().ref_precondition(self._h, self._dt(y), layout, _ptr(y), _ptr(x), self.workers))
        return x

    def fused_spmv(self, u, p, q, z, alpha, beta, layout=0):
        u, p, q, z = (np.array(a, copy=True, order="C") for a in (u, p, q, z))
        sg = C.c_double()
        _check(ref_lib().ref_fused_spmv(self._h, self._dt(u), layout, _ptr(u), _ptr(p), _ptr(q),
                                        _ptr(z), float(alpha), float(beta), C.byref(sg), self.workers))
        return u, p, q, sg.value

    def fused_prec(self, r, q, alpha, layout=0):
        r = np.array(r, copy=True, order="C")
        q = np.ascontiguousarray(q)
        z = np.zeros_like(r)
        rn, ka = C.c_double(), C.c_double()
        _check(ref_lib().ref_fused_prec(self._h, self._dt(r), layout, _ptr(r), _ptr(z), _ptr(q),
                                        float(alpha), C.byref(rn), C.byref(ka), self.workers))
        return r, z, rn.value, ka.value

    def dot(self, x, y, layout=0):
        out = C.c_double()
        _check(ref_lib().ref_dot(self._h, self._dt(x), layout, _ptr(np.ascontiguousarray(x)),
                                 _ptr(np.ascontiguousarray(y)), C.byref(out), self.workers))
        return out.value

    def nrm2(self, x, layout=0):
        out = C.c_double()
        _check(ref_lib().ref_nrm2(self._h, self._dt(x), layout, _ptr(np.ascontiguousarray(x)),
                                  C.byref(out), self.workers))
        return out.value

    def true_residual(self, u, f, layout=0):
        out = C.c_double()
        _check(ref_lib().ref_true_residual(self._h, self._dt(u), layout, _ptr(np.ascontiguousarray(u)),
                                           _ptr(np.ascontiguousarray(f)), C.byref(out), self.workers))
        return out.value

    def solve(self, f, u0=None, epsilon=1e-5, tau=1e-20, maxiter=500, variant="interleaved", layout=0,
              backend="matrix-free"):
        f = np.ascontiguousarray(f)
        u = np.empty_like(f)
        cap = maxiter + 2
        hs = [np.zeros(cap) for _ in range(4)]
        res = _RefResult()
        if backend == "csr" and variant != "standard":
            raise ValueError("SolverConfig: the interleaved variant exists for the matrix-free "
                             "backend only")
        code = 2 if backend == "csr" else (1 if variant == "interleaved" else 0)
        _check(ref_lib().ref_solve(self._h, self._dt(f), layout, _ptr(f),
                                   _ptr(np.ascontiguousarray(u0) if u0 is not None else None),
                                   epsilon, tau, maxiter, code,
                                   self.workers, _ptr(u), C.byref(res), *hs))
        t = {k: getattr(res, k) for k in ("fused_prec_s", "fused_spmv_s", "spmv_s", "prec_s",
                                          "blas_s", "setup_s", "total_s")}
        return u, Result(res.iterations, bool(res.converged), res.true_residual,
                         hs[0][:res.n_residual].copy(), hs[1][:res.n_kappa].copy(),
                         hs[2][:res.n_alpha].copy(), hs[3][:res.n_beta].copy(), 0, t)


def ref_panel(m, sphere=True, extent=2.0):
    area, diag = np.empty((m, m)), np.empty((m, m))
    east, north = np.empty((max(m - 1, 0), m)), np.empty((m, max(m - 1, 0)))
    _check(ref_lib().ref_panel(0 if sphere else 1, m, extent, _ptr(area), _ptr(east), _ptr(north), _ptr(diag)))
    return area, east, north, diag


def ref_vertical_grid(n_z, h):
    r = np.empty(n_z + 1)
    _check(ref_lib().ref_vertical_grid(n_z, h, r))
    return r


def ref_profile(n_z, h, omega2, lambda2):
    out = [np.empty(n_z) for _ in range(4)]
    _check(ref_lib().ref_profile(n_z, h, omega2, lambda2, *out))
    return tuple(out)
