"""Worker for tests/test_variants.py: one process per kernel-variant setting.

The launch-mode switches (ACG_PDL, ACG_CONSUME, ACG_KSPLIT) are read once per
process, so each setting runs in its own process. It runs the fused sweeps, apply,
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
    # the step API in uneven batches (graph chunks, direct remainders, the
    # consumed-reduction flush at every batch end) against one oracle solve
    from paper_1302_7193_b200 import capi
    cc = capi.Context(o.ap, o.bp, o.cp, o.d, o.area, o.east, o.north, o.diag,
                      dtype=capi.F32 if dtype == np.float32 else capi.F64)
    fd = cc.field().upload(f)
    sv = capi.Solver(cc, epsilon=1e-300, tau=1e-300, maxiter=41)
    sv.start(fd)
    for n in (5, 17, 3, 16):
        sv.iterate(n)
    rs = sv.finish()
    _, ro = o.solve(f, epsilon=1e-300, tau=1e-300, maxiter=41)
    ok = rs["iterations"] == ro.iterations and all(
        np.array_equal(rs[h], getattr(ro, h))
        for h in ("residual_history", "kappa_history", "alpha_history", "beta_history"))
    sv.close()
    fd.close()
    cc.close()
    if not ok:
        return "step API batches"
    return None


# (m, n_z) reaching every shipped kernel: even / ragged widths (pair and quad
# kernels, TMEM sweeps), odd m (k_fused_spmv_tile; k_thomas_tm for fp32), fp64
# columns whose z' needs all 512 TMEM columns (one CTA per SM: n_z 160), and
# columns taller than TMEM holds (k_thomas, z' in global memory: fp64 n_z 272,
# fp32 n_z 520)
# and power-of-two panels m < 512 whose K2 splits the levels over 512/m thread
# groups in one CTA (fp64: 8, 4, 2 groups, ragged last group) with the
# consumed-reduction prologues
SHAPES = ((128, 24), (66, 19), (65, 12), (32, 160), (16, 272), (8, 520), (64, 13), (256, 33))


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
