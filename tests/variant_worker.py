"""Worker for tests/test_variants.py: one process per kernel-variant setting.

The launch-mode switch ACG_PDL is read once per process,
so each setting runs in its own process. It runs the fused sweeps, apply,
precondition and two full solves (fp64 and fp32, over SHAPES) and compares them bit for bit with the CPU oracle.
Prints VARIANT_OK or the first mismatch.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_1302_7193_b200 as acg  # noqa: E402
from oracle.oracle import Oracle, Problem  # noqa: E402


def check(m, n_z, dtype):
    prob = Problem(m, n_z, True)
    o = Oracle(prob)
    g = acg.vertical_grid(prob.n_z, prob.h)
    pro = acg.vertical_profile(g, prob.omega2, prob.lambda2)
    cls = acg.OperatorContextF32 if dtype == np.float32 else acg.OperatorContext
    ctx = cls(pro, acg.cubed_sphere_panel(prob.m))
    x = o.random_field(5, dtype)
    if not np.array_equal(acg.apply(ctx, x), o.apply(x)):
        return "apply"
    if not np.array_equal(acg.precondition(ctx, x), o.precondition(x)):
        return "precondition"
    u, p, q, z = (o.random_field(s, dtype) for s in (101, 104, 105, 103))
    gu, gp, gq, gs = acg.interleaved_spmv_kernel(ctx, u, p, q, z, 0.37, 0.21)
    ou, op, oq, osg, _ = o.fused_spmv(u, p, q, z, 0.37, 0.21)
    if not (np.array_equal(gu, ou) and np.array_equal(gp, op) and np.array_equal(gq, oq)
            and gs == osg):
        return "interleaved_spmv_kernel"
    r = o.random_field(102, dtype)
    gr, gz, grn, gk = acg.interleaved_prec_kernel(ctx, r, q, 0.37)
    orr, oz, orn, ok, _, _ = o.fused_prec(r, q, 0.37)
    if not (np.array_equal(gr, orr) and np.array_equal(gz, oz) and grn == orn and gk == ok):
        return "interleaved_prec_kernel"
    f = o.random_field(42, dtype)
    ug, rg = acg.solve(ctx, f, epsilon=1e-9 if dtype == np.float64 else 1e-4, maxiter=60)
    uo, ro = o.solve(f, epsilon=1e-9 if dtype == np.float64 else 1e-4, maxiter=60)
    if rg.iterations != ro.iterations:
        return f"iterations {rg.iterations} vs {ro.iterations}"
    for h in ("residual_history", "kappa_history", "alpha_history", "beta_history"):
        if not np.array_equal(getattr(rg, h), getattr(ro, h)):
            return h
    if not np.array_equal(ug, uo):
        return "solution"
    return None


# (m, n_z) reaching every shipped kernel: even / ragged widths (pair and quad
# kernels, TMEM sweeps), odd m (k_fused_spmv_tile; k_thomas_tm for fp32), fp64
# columns whose z' needs all 512 TMEM columns (one CTA per SM: n_z 160), and
# columns taller than TMEM holds (k_thomas, z' in global memory: fp64 n_z 272,
# fp32 n_z 520)
SHAPES = ((128, 24), (66, 19), (65, 12), (32, 160), (16, 272), (8, 520))


def main():
    for m, n_z in SHAPES:
        for dt in (np.float64, np.float32):
            bad = check(m, n_z, dt)
            if bad:
                print(f"VARIANT_MISMATCH m={m} n_z={n_z} {np.dtype(dt).name}: {bad}", flush=True)
                return
    print("VARIANT_OK", flush=True)


if __name__ == "__main__":
    main()
