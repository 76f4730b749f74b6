"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Run in the build container (needs oracle/_ref, i.e. the reference compiled from
/root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Every array here is the output of the unmodified reference hot path
(proj/include/anisocg/*.hpp + src/grid.cpp + src/profile.cpp) called through
oracle/ref_harness.cpp. The fixtures travel with the repo so the oracle and the
GPU path are pinned to the reference even where /root/reference is absent.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import (Problem, Reference, ref_panel, ref_profile,  # noqa: E402
                           ref_vertical_grid)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {}
    # ---- setup (grid.cpp, profile.cpp)
    out["grid_4_0.1"] = ref_vertical_grid(4, 0.1)
    out["grid_128_0.01"] = ref_vertical_grid(128, 0.01)
    for m in (1, 2, 4, 8, 13):
        for sphere in (True, False):
            a, e, n, d = ref_panel(m, sphere, 2.0)
            tag = f"{'sphere' if sphere else 'planar'}_{m}"
            out[f"panel_{tag}_area"], out[f"panel_{tag}_east"] = a, e
            out[f"panel_{tag}_north"], out[f"panel_{tag}_diag"] = n, d
    for n_z, h, om, la in ((2, 0.1, 1.0, 1.0), (16, 0.02, 6.71e-4, 3.32e-2), (64, 1e-2, 6.71e-4, 3.32e-2),
                           (12, 0.05, 0.3, 0.7)):
        ap, bp, cp, dd = ref_profile(n_z, h, om, la)
        tag = f"{n_z}_{h}_{om}_{la}"
        out[f"prof_{tag}_ap"], out[f"prof_{tag}_bp"] = ap, bp
        out[f"prof_{tag}_cp"], out[f"prof_{tag}_d"] = cp, dd

    # ---- operators and fused sweeps (operator.hpp)
    for (m, n_z, sphere) in ((4, 8, True), (8, 16, True), (8, 16, False), (13, 7, True), (1, 12, True)):
        prob = Problem(m, n_z, sphere)
        ref = Reference(prob)
        tag = f"{m}_{n_z}_{'s' if sphere else 'p'}"
        for dt, dn in ((np.float64, "f64"), (np.float32, "f32")):
            x = ref.random_field(5, dt)
            out[f"op_{tag}_{dn}_x"] = x
            out[f"op_{tag}_{dn}_apply"] = ref.apply(x)
            out[f"op_{tag}_{dn}_prec"] = ref.precondition(x)
            u, p, q, z, r = (ref.random_field(s, dt) for s in (101, 104, 105, 103, 102))
            u2, p2, q2, sg = ref.fused_spmv(u, p, q, z, 0.37, 0.21)
            out[f"op_{tag}_{dn}_spmv_u"], out[f"op_{tag}_{dn}_spmv_p"] = u2, p2
            out[f"op_{tag}_{dn}_spmv_q"], out[f"op_{tag}_{dn}_spmv_sigma"] = q2, np.array(sg)
            r2, z2, rn, ka = ref.fused_prec(r, q, 0.37)
            out[f"op_{tag}_{dn}_prec2_r"], out[f"op_{tag}_{dn}_prec2_z"] = r2, z2
            out[f"op_{tag}_{dn}_prec2_rk"] = np.array([rn, ka])
            out[f"op_{tag}_{dn}_dot"] = np.array([ref.dot(u, p), ref.nrm2(u), ref.true_residual(u, r)])

    # ---- solves (solver.hpp)
    cases = [
        ("s8_16_il", Problem(8, 16), np.float64, dict(epsilon=1e-8, maxiter=300, variant="interleaved")),
        ("s8_16_std", Problem(8, 16), np.float64, dict(epsilon=1e-8, maxiter=300, variant="standard")),
        ("s8_16_f32", Problem(8, 16), np.float32, dict(epsilon=1e-4, maxiter=200, variant="interleaved")),
        ("p4_8_std5", Problem(4, 8, False), np.float64, dict(epsilon=1e-300, maxiter=5, variant="standard")),
        ("s16_32_court", Problem(16, 32, True, 6.71e-4 * 16 ** 2), np.float64,
         dict(epsilon=1e-300, maxiter=50, variant="interleaved")),
        ("s1_16_il", Problem(1, 16), np.float64, dict(variant="interleaved")),
        ("s8_16_exh", Problem(8, 16), np.float64, dict(epsilon=1e-300, maxiter=3, variant="interleaved")),
    ]
    for tag, prob, dt, kw in cases:
        ref = Reference(prob)
        f = ref.random_field(13 if tag.startswith("s1_") else 42, dt)
        u, res = ref.solve(f, **kw)
        out[f"solve_{tag}_u"] = u
        out[f"solve_{tag}_res"] = res.residual_history
        out[f"solve_{tag}_kap"] = res.kappa_history
        out[f"solve_{tag}_alp"] = res.alpha_history
        out[f"solve_{tag}_bet"] = res.beta_history
        out[f"solve_{tag}_meta"] = np.array([res.iterations, int(res.converged), res.true_residual])

    # ---- BASELINE config 1: 128x128x64 fp64, eps = 1e-10 (all cores)
    prob = Problem(128, 64)
    ref = Reference(prob, workers=os.cpu_count() or 1)
    f = ref.random_field(42)
    u, res = ref.solve(f, epsilon=1e-10, maxiter=500)
    out["c1_f_sha"] = np.array(sha(f))
    out["c1_u_sha"] = np.array(sha(u))
    out["c1_u_sample"] = u.reshape(-1)[::997].copy()
    out["c1_res"], out["c1_kap"] = res.residual_history, res.kappa_history
    out["c1_alp"], out["c1_bet"] = res.alpha_history, res.beta_history
    out["c1_meta"] = np.array([res.iterations, int(res.converged), res.true_residual])
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print(f"wrote {len(out)} arrays; C1 iterations = {res.iterations}")


if __name__ == "__main__":
    main()
