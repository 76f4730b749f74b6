"""Device-resident edge of the ``anisocg`` API.

``solve``, ``apply`` and ``precondition`` accept CUDA arrays (torch tensors or
anything exposing ``__cuda_array_interface__``) of the reference's shapes —
(m, m, n_z) ``layout="vertical"`` or (m, n_z, m) ``"horizontal"`` — and return
CUDA arrays of the same kind. The field never crosses PCIe: the relayout to
the device's plane-major storage runs on the GPU (acg_field_upload_device /
acg_field_download_device, include/acg.h), so a GPU-resident caller pays only
the solve. Results are the same bits as the host path (tests/test_gpu_parity.py).
Host numpy arrays keep going through the reference-compatible ``_anisocg``
module unchanged (paper_1302_7193_b200/__init__.py routes by argument type).
"""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np

from . import capi

_LAYOUTS = {"vertical": capi.VERTICAL, "horizontal": capi.HORIZONTAL}


def _layout(name):
    try:
        return _LAYOUTS[name]
    except KeyError:
        raise ValueError("layout must be 'vertical' or 'horizontal'") from None


def _empty_like(a):
    """A new CUDA array of a's kind, shape and dtype (torch, else CuPy)."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return torch.empty_like(a, memory_format=torch.contiguous_format)
    except ImportError:  # pragma: no cover - torch is part of this image
        pass
    try:
        import cupy  # noqa: F401  (optional)
        return cupy.empty_like(a)
    except ImportError as exc:
        raise TypeError("device arrays must be torch tensors or CuPy arrays") from exc


class _Ctx:
    """capi view of an anisocg.OperatorContext (borrowed acg_context)."""

    def __init__(self, ctx):
        self.view = capi.Context.borrow(ctx._handle, owner=ctx)

    def field(self, a=None, layout=capi.VERTICAL):
        f = self.view.field()
        if a is not None:
            f.upload(a, layout)
        return f


def apply(ctx, x, workers=1, *, layout="vertical"):
    """y = A x (operator.hpp:101-135) for a CUDA array x; returns a CUDA array."""
    L = _layout(layout)
    c = _Ctx(ctx)
    fx, fy = c.field(x, L), c.field()
    capi.apply(c.view, fx, fy)
    return fy.download(L, out=_empty_like(x))


def precondition(ctx, y, workers=1, *, layout="vertical"):
    """x = M^-1 y (operator.hpp:141-191) for a CUDA array y; returns a CUDA array."""
    L = _layout(layout)
    c = _Ctx(ctx)
    fy, fx = c.field(y, L), c.field()
    capi.precondition(c.view, fy, fx)
    return fx.download(L, out=_empty_like(y))


def solve(ctx, f, u0=None, epsilon=1e-5, tau=1e-20, maxiter=500, variant="interleaved",
          backend="matrix-free", workers=1, *, layout="vertical"):
    """solve() (solver.hpp:373-378) with CUDA arrays in and out; same defaults and
    argument errors as the host binding. Returns (u, result) where result has the
    SolveResult attributes (iterations, converged, true_residual, *_history, timings)."""
    if variant not in ("standard", "interleaved"):
        raise ValueError("variant must be 'standard' or 'interleaved'")
    if backend not in ("matrix-free", "csr"):
        raise ValueError("backend must be 'matrix-free' or 'csr'")
    # SolverConfig::validate (solver.hpp:27-35): the same checks and messages as
    # the host path
    if not (epsilon > 0):
        raise ValueError("SolverConfig: epsilon must be > 0")
    if not (tau > 0):
        raise ValueError("SolverConfig: tau must be > 0")
    if maxiter < 1:
        raise ValueError("SolverConfig: maxiter must be >= 1")
    if workers < 1:
        raise ValueError("SolverConfig: workers must be >= 1")
    L = _layout(layout)
    c = _Ctx(ctx)
    ff = c.field(f, L)
    fu0 = c.field(u0, L) if u0 is not None else None
    fu = c.field()
    r = capi.solve(c.view, ff, u0=fu0, u_out=fu, epsilon=epsilon, tau=tau, maxiter=maxiter,
                   variant=capi.STANDARD if variant == "standard" else capi.INTERLEAVED,
                   backend=capi.CSR if backend == "csr" else capi.MATRIX_FREE, layout=L)
    u = fu.download(L, out=_empty_like(f))
    res = SimpleNamespace(
        iterations=r["iterations"], converged=r["converged"], true_residual=r["true_residual"],
        residual_history=np.asarray(r["residual_history"]),
        kappa_history=np.asarray(r["kappa_history"]),
        alpha_history=np.asarray(r["alpha_history"]),
        beta_history=np.asarray(r["beta_history"]),
        timings=SimpleNamespace(**r["timings"]), kernel_launches=r["kernel_launches"])
    return u, res
