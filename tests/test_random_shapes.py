"""Seeded random shapes through the whole solve, bit-exact against the CPU
oracle: every kernel-selection boundary (odd / even / power-of-two m, narrow
and wide panels, TMEM and global-memory columns, 1 and 2 slabs, both
precisions, both loops) is crossed by some draw, not only the hand-picked
shapes of test_gpu_parity.py. The draws are fixed (seed 20261017), so a
failure names a reproducible (m, n_z, ...) case.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle, Problem

pytestmark = pytest.mark.gpu


def draws(n=28, seed=20261017):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        m = int(rng.choice([rng.integers(1, 40), rng.integers(40, 300), 2 ** rng.integers(3, 9)]))
        n_z = int(rng.choice([rng.integers(1, 16), rng.integers(16, 140), rng.integers(250, 300)]))
        dtype = np.float32 if rng.random() < 0.35 else np.float64
        variant = "standard" if rng.random() < 0.3 else "interleaved"
        sphere = bool(rng.random() < 0.7)
        slabs = 2 if (m >= 4 and rng.random() < 0.25) else 1
        out.append((i, m, n_z, dtype, variant, sphere, slabs))
    return out


@pytest.mark.parametrize("case", draws(), ids=lambda c: f"{c[0]}-m{c[1]}-nz{c[2]}-"
                         f"{np.dtype(c[3]).name}-{c[4]}-{'sph' if c[5] else 'pl'}-s{c[6]}")
def test_random_shape_solve_bit_exact(acg, case):
    _, m, n_z, dtype, variant, sphere, slabs = case
    prob = Problem(m, n_z, sphere)
    o = Oracle(prob)
    g = acg.vertical_grid(prob.n_z, prob.h)
    pro = acg.vertical_profile(g, prob.omega2, prob.lambda2)
    pan = acg.cubed_sphere_panel(m) if sphere else acg.planar_panel(m, prob.extent)
    cls = acg.OperatorContextF32 if dtype == np.float32 else acg.OperatorContext
    ctx = cls(pro, pan, slabs=slabs)
    f = o.random_field(42, dtype)
    kw = dict(epsilon=1e-4 if dtype == np.float32 else 1e-9, maxiter=30, variant=variant)
    u, r = acg.solve(ctx, f, **kw)
    uo, ro = o.solve(f, **kw)
    assert r.iterations == ro.iterations
    exact = ctx.info["exact_tree"] if slabs > 1 else True
    for h in ("residual_history", "kappa_history", "alpha_history", "beta_history"):
        a, b = getattr(r, h), getattr(ro, h)
        if exact:
            assert np.array_equal(a, b), h
        else:  # non-tree slabs: the documented pairwise combination of slab sums
            assert np.allclose(a, b, rtol=1e-10 if dtype == np.float64 else 1e-5, atol=0), h
    if exact:
        assert np.array_equal(u, uo)
