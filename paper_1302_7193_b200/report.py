"""Report and wire formats of the reference.

* ``residual_csv`` / ``cost_model_csv`` / ``geometry_csv`` / ``dump_field`` — the
  text (bytes) of proj/include/anisocg/io.hpp, produced by the B200 build's own
  io.cpp (include/anisocg/io.hpp) and pinned byte for byte to the reference's
  writers (tests/test_report.py).
* ``solve_json`` — the object the reference CLI prints for ``solve``
  (proj/tools/main.cpp:140-162), from a solve's arguments and result.
* ``BENCH_CSV_HEADER`` / ``bench_csv_row`` — the reference CLI's bench CSV schema
  (main.cpp:270-281), filled from one timed solve (time per iteration and the
  paper's cost model for the GFLOP/s and GB/s estimates, main.cpp:231-247).
"""
from __future__ import annotations

from . import _anisocg as _ext

residual_csv = _ext.residual_csv
cost_model_csv = _ext.cost_model_csv
geometry_csv = _ext.geometry_csv
dump_field = _ext.dump_field

BENCH_CSV_HEADER = ("backend,variant,layout,precision,workers,m,nz,iters,setup_ms,"
                    "time_per_iter_ms,spmv_ms,prec_ms,blas_ms,fused_spmv_ms,fused_prec_ms,"
                    "gflops_est,gbs_est")


def write(path, text):
    """Write a report string (or dump bytes) to `path`."""
    mode = "wb" if isinstance(text, (bytes, bytearray)) else "w"
    with open(path, mode, **({} if mode == "wb" else {"newline": "\n"})) as fh:
        fh.write(text)


def _timings(t):
    get = (lambda k: t[k]) if isinstance(t, dict) else (lambda k: getattr(t, k))
    keys = ("spmv", "prec", "blas", "fused_spmv", "fused_prec", "setup", "total")
    return {f"{k}_s": get(k) for k in keys}


def solve_json(result, *, geometry="cubed-sphere", m, nz, h_atmos, omega2, lambda2,
               backend="matrix-free", variant="interleaved", layout="vertical",
               precision="double", epsilon=1e-5, tau=1e-20, maxiter=500, workers=1, seed=42,
               extent=None):
    """The reference CLI's solve report (main.cpp:140-162) as a dict."""
    h = list(result.residual_history)
    r0, rl = (h[0], h[-1]) if h else (0.0, 0.0)
    out = {"geometry": geometry, "m": m, "nz": nz, "h_atmos": h_atmos, "omega2": omega2,
           "lambda2": lambda2, "backend": backend, "variant": variant, "layout": layout,
           "precision": precision, "epsilon": epsilon, "tau": tau, "maxiter": maxiter,
           "workers": workers, "seed": seed, "rhs": "splitmix64-uniform",
           "iterations": result.iterations, "converged": bool(result.converged),
           "residual0": r0, "residual": rl, "rel_residual": rl / r0 if r0 > 0 else 0.0,
           "true_residual": result.true_residual, "timings": _timings(result.timings)}
    if geometry == "planar":
        out["extent"] = extent
    return out


def bench_csv_row(result, *, iters, m, nz, backend="matrix-free", variant="interleaved",
                  layout="vertical", precision="double", workers=1):
    """One row of the reference bench CSV from a fixed-iteration solve's timings."""
    t = _timings(result.timings)
    per_iter = (t["total_s"] - t["setup_s"]) / iters
    kernel = "interleaved_total" if variant == "interleaved" else "pcg_total"
    flops, refs = _ext.cost_model(kernel, "none")
    n = m * m * nz
    s = 4 if precision == "single" else 8
    vals = [t["setup_s"] * 1e3, per_iter * 1e3] + [t[k] / iters * 1e3 for k in
                                                  ("spmv_s", "prec_s", "blas_s", "fused_spmv_s",
                                                   "fused_prec_s")]
    est = [flops * n / per_iter * 1e-9, refs * n * s / per_iter * 1e-9] if per_iter > 0 else [0.0, 0.0]
    fmt = lambda v: f"{v:.6g}"  # noqa: E731  (ostream precision 6)
    return ",".join([backend, variant, layout, precision, str(workers), str(m), str(nz),
                     str(iters)] + [fmt(v) for v in vals + est])
