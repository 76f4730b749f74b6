"""The reference's acceptance gate (proj/tests/acceptance_main.cpp)
criteria that concern the hot path, run on the GPU build.

* criterion 5 (acceptance_main.cpp:308-339): 256x256x128 cubed sphere, RHS seed
  42, interleaved PCG converges to 1e-5 in <= 100 iterations; seeds 1-5 in
  <= 120 — and the seed-42 solve is bit-identical to the reference run here;
* criterion 7 (:405-431): iteration counts for m in {32, 64, 128}, n_z = 64,
  omega^2 Courant-scaled from the m = 256 value. The reference's gate asks for
  a spread <= 25%; the reference itself (oracle/_ref, run here) takes 59, 69
  and 76 iterations, a 28.8% spread, so the GPU build is held to the
  reference's own counts (it takes the same, bit-identical solves) and the
  spread is reported;
* criterion 8 (:435-477): determinism — the reference checks 1 vs N OpenMP
  workers; here repeated runs and 1 vs 2/4 slabs (tree-aligned) are
  bit-identical;
* criterion 9 (:481-521): directional performance — matrix-free standard
  faster than the CSR backend, interleaved no slower than standard, per
  iteration from the solve's own timings (total - setup, median of 5 after a
  warm-up), at 512^2 x 128 (the reference's 64^3 case is launch-bound on a GPU:
  a few microseconds per kernel).
"""
import os

import numpy as np
import pytest

from oracle.oracle import Problem, Reference, ref_available

pytestmark = pytest.mark.gpu


def ctx_for(acg, m, n_z, omega2=6.71e-4, slabs=1):
    g = acg.vertical_grid(n_z, 1e-2)
    return acg.OperatorContext(acg.vertical_profile(g, omega2, 3.32e-2),
                               acg.cubed_sphere_panel(m), slabs=slabs)


def test_criterion5_reference_convergence(acg):
    ctx = ctx_for(acg, 256, 128)
    f = acg.random_field(256, 128, 42)
    u, r = acg.solve(ctx, f, epsilon=1e-5, maxiter=100, variant="interleaved")
    assert r.converged and r.iterations <= 100
    if ref_available():
        ref = Reference(Problem(256, 128), workers=os.cpu_count() or 1)
        uo, ro = ref.solve(f, epsilon=1e-5, maxiter=100, variant="interleaved")
        assert r.iterations == ro.iterations == 79  # SURVEY §6 probe
        assert np.array_equal(r.residual_history, ro.residual_history)
        assert np.array_equal(u, uo)
    for seed in (1, 2, 3, 4, 5):
        _, ra = acg.solve(ctx, acg.random_field(256, 128, seed), epsilon=1e-5, maxiter=120,
                          variant="interleaved")
        assert ra.converged and ra.iterations <= 120, (seed, ra.iterations)


def test_criterion7_grid_robust_iterations(acg):
    iters, ref_iters = [], []
    for m in (32, 64, 128):
        scale = 256.0 / m
        omega2 = 6.71e-4 * scale * scale
        ctx = ctx_for(acg, m, 64, omega2=omega2)
        f = acg.random_field(m, 64, 42)
        _, r = acg.solve(ctx, f, epsilon=1e-5, maxiter=500, variant="interleaved")
        iters.append(r.iterations if r.converged else 501)
        if ref_available():
            ref = Reference(Problem(m, 64, True, omega2), workers=os.cpu_count() or 1)
            _, ro = ref.solve(f, epsilon=1e-5, maxiter=500, variant="interleaved")
            assert np.array_equal(r.residual_history, ro.residual_history), m
            ref_iters.append(ro.iterations)
    assert iters == (ref_iters or [59, 69, 76])
    spread = (max(iters) - min(iters)) / min(iters)
    print(f"criterion 7 iterations {iters}, spread {spread:.1%} (reference gate: <= 25%)")


def test_criterion8_determinism(acg):
    f = acg.random_field(128, 64, 42)
    base = None
    for slabs in (1, 1, 2, 4):
        ctx = ctx_for(acg, 128, 64, slabs=slabs)
        assert ctx.info["exact_tree"]
        u, r = acg.solve(ctx, f, epsilon=1e-10, maxiter=300)
        if base is None:
            base = (u, r)
            continue
        assert r.iterations == base[1].iterations
        assert np.array_equal(r.residual_history, base[1].residual_history)
        assert np.array_equal(u, base[0])


def _per_iter(acg, ctx, f, variant, backend, iters=25, reps=5):
    acg.solve(ctx, f, epsilon=1e-300, tau=1e-300, maxiter=1, variant=variant, backend=backend)
    times = []
    for _ in range(reps):
        _, r = acg.solve(ctx, f, epsilon=1e-300, tau=1e-300, maxiter=iters, variant=variant,
                         backend=backend)
        times.append((r.timings.total_s - r.timings.setup_s) / iters)
    return sorted(times)[reps // 2]


def test_criterion9_directional_performance(acg):
    ctx = ctx_for(acg, 512, 128)
    f = acg.random_field(512, 128, 42)
    t_std = _per_iter(acg, ctx, f, "standard", "matrix-free")
    t_csr = _per_iter(acg, ctx, f, "standard", "csr")
    t_il = _per_iter(acg, ctx, f, "interleaved", "matrix-free")
    ctx.release_scratch()
    print(f"per-iteration ms: matrix-free standard {t_std * 1e3:.3f}, csr {t_csr * 1e3:.3f}, "
          f"interleaved {t_il * 1e3:.3f}")
    assert t_std < t_csr
    assert t_il <= t_std
