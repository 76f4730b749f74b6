"""B200-native matrix-free PCG for the anisotropic 3D pressure-correction
equation (arXiv 1302.7193), a drop-in for the reference's ``anisocg`` module.

Everything numerical runs in hand-written sm_100a kernels in ``libacg_cuda.so``
behind the C ABI of ``include/acg.h``; ``_anisocg`` is the reference's Python
surface (proj/python/bindings.cpp) over the host C++ shim. There is no CPU
fallback: importing this package without its built extension fails loudly, and
every compute call fails with a CUDA error on a machine without a GPU.
"""
import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from ._anisocg import (  # noqa: F401
        KernelTimings,
        OperatorContext,
        OperatorContextF32,
        PanelGeometry,
        SolveResult,
        VerticalGrid,
        VerticalProfile,
        anisotropy,
        apply,
        assemble_csr,
        axpy,
        cost_model,
        cubed_sphere_panel,
        dot,
        interleaved_prec_kernel,
        interleaved_spmv_kernel,
        kernel_launch_count,
        nrm2,
        planar_panel,
        precondition,
        random_field,
        release_scratch,
        scal,
        solve,
        true_residual,
        vertical_grid,
        vertical_profile,
    )
except ImportError as exc:  # pragma: no cover - the product must not run without its CUDA build
    raise ImportError(
        "paper_1302_7193_b200: the CUDA extension is not built "
        f"({exc}); run `make` (or __graft_entry__.build()) first") from exc

LIBRARY_PATH = _os.path.join(_HERE, "libacg_cuda.so")

from . import _anisocg as _ext  # noqa: E402
from . import capi as _capi  # noqa: E402
from . import device as _device  # noqa: E402


def solve(ctx, f, *args, **kw):
    """solve(ctx, f, u0=None, epsilon=1e-5, tau=1e-20, maxiter=500, variant="interleaved",
    backend="matrix-free", workers=1, *, layout="vertical") -> (u, SolveResult).
    Host (numpy) arrays: the reference binding (bindings.cpp:204-237). CUDA arrays
    (torch, CuPy): device-resident, no PCIe transfer (device.solve)."""
    if _capi.is_cuda_array(f):
        return _device.solve(ctx, f, *args, **kw)
    return _ext.solve(ctx, f, *args, **kw)


def apply(ctx, x, *args, **kw):
    """y = A x; numpy in/out (reference binding) or CUDA arrays in/out (device.apply)."""
    if _capi.is_cuda_array(x):
        return _device.apply(ctx, x, *args, **kw)
    return _ext.apply(ctx, x, *args, **kw)


def precondition(ctx, y, *args, **kw):
    """x = M^-1 y; numpy in/out (reference binding) or CUDA arrays in/out (device.precondition)."""
    if _capi.is_cuda_array(y):
        return _device.precondition(ctx, y, *args, **kw)
    return _ext.precondition(ctx, y, *args, **kw)

__all__ = [
    "KernelTimings", "OperatorContext", "OperatorContextF32", "PanelGeometry", "SolveResult",
    "VerticalGrid", "VerticalProfile", "anisotropy", "apply", "assemble_csr", "axpy",
    "cost_model", "cubed_sphere_panel", "dot", "interleaved_prec_kernel",
    "interleaved_spmv_kernel", "kernel_launch_count", "nrm2", "planar_panel", "precondition",
    "random_field", "release_scratch", "scal", "solve", "true_residual", "vertical_grid", "vertical_profile",
]
