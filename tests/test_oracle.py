"""Pin the CPU oracle (oracle/acg_oracle.c) before trusting it (CPU-only).

1. the reference's own known-answer values (proj/tests/test_grid.cpp,
   test_profile.cpp, test_field.cpp), asserted at the reference's tolerances;
2. the golden fixtures generated from the reference itself
   (tests/golden/make_golden.py) — bit for bit;
3. the reference compiled from source (oracle/_ref), when present — bit for
   bit on fresh random cases.
"""
import hashlib
import math
import os

import numpy as np
import pytest

from oracle.oracle import (Oracle, Problem, Reference, anisotropy, panel, ref_available,
                           vertical_grid, vertical_profile)

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------ known answers
def test_grid_known_answers():
    g = vertical_grid(4, 0.1)  # test_grid.cpp:16-24
    np.testing.assert_allclose(g[1:4], [1.00625, 1.025, 1.05625], rtol=1e-15)
    assert g[0] == 1.0 and g[4] == 1.1
    e = vertical_grid(1, 0.01)
    assert e[0] == 1.0 and e[1] == 1.01
    dz = np.diff(vertical_grid(128, 0.01))  # test_grid.cpp:29-43
    assert math.isclose(dz.min(), 6.103515625e-07, rel_tol=1e-9)
    assert math.isclose(dz.max(), 1.5563964843750002e-04, rel_tol=1e-9)


def test_panel_known_answers():
    area, east, north, diag = panel(4, True)  # test_grid.cpp:86-102
    assert math.isclose(area[0, 0], 0.081455587595345325, rel_tol=1e-13)
    assert math.isclose(area[1, 1], 0.2013579207903308, rel_tol=1e-13)
    assert math.isclose(area[2, 1], 0.2013579207903308, rel_tol=1e-13)
    assert math.isclose(east[1, 1], 0.97429061355337199, rel_tol=1e-13)
    assert math.isclose(north[0, 0], 0.90137534005291164, rel_tol=1e-13)
    assert math.isclose(panel(2, True)[1][0, 0], 0.93380979565807565, rel_tol=1e-13)
    assert math.isclose(panel(1, True)[0][0, 0], 4 * math.pi / 6, rel_tol=1e-12)
    for m in (2, 5, 16, 64):  # areas partition the sixth-sphere (:76-84)
        a = panel(m, True)[0]
        assert abs(a.sum() - 4 * math.pi / 6) / (4 * math.pi / 6) <= 1e-12
    np.testing.assert_array_equal(panel(3, False, 3.0)[3], [[2, 3, 2], [3, 4, 3], [2, 3, 2]])
    a1 = panel(1, False, 5.0)
    assert a1[3][0, 0] == 0.0 and a1[0][0, 0] == 25.0


def test_profile_known_answers():
    ap, bp, cp, d = vertical_profile(vertical_grid(2, 0.1), 1.0, 1.0)  # test_profile.cpp:29-39
    assert math.isclose(d[0], -0.02563020833333322, rel_tol=1e-14)
    assert math.isclose(d[1], -0.084703125000000254, rel_tol=1e-14)
    assert math.isclose(ap[0], -1.0, rel_tol=1e-15)
    assert math.isclose(bp[0], 819.83336720179102, rel_tol=1e-13)
    assert math.isclose(bp[0] * d[0], -21.012499999999978, rel_tol=1e-14)
    assert math.isclose(cp[1], 248.0723113816629, rel_tol=1e-13)
    ap, bp, cp, d = vertical_profile(vertical_grid(8, 0.1), 2.0, 0.5)
    assert cp[0] == 0.0 and bp[7] == 0.0 and np.all(d != 0)
    ap, bp, cp, d = vertical_profile(vertical_grid(16, 0.02), 6.71e-4, 3.32e-2)
    np.testing.assert_allclose(ap, -1.0 / 6.71e-4, rtol=1e-15)


def test_anisotropy_known_answer():
    area = panel(256, False, 2.0)[0]  # test_grid.cpp:137-152
    g2 = anisotropy(area, vertical_grid(128, 0.01), 3.32e-2)
    col = g2[0, 0]
    assert math.isclose(col.max(), 5439488.0017414093, rel_tol=1e-12)
    assert col.min() > 80.0


def test_linear_index_examples():
    # test_field.cpp:11-16 : l(1,2,3) on 16x16x128
    m, n_z = 16, 128
    assert n_z * (m * 1 + 2) + 3 == 2307
    assert m * (n_z * 2 + 3) + 1 == 4145
    o = Oracle(Problem(4, 3))
    v, h = o.random_field(99, layout=0), o.random_field(99, layout=1)
    np.testing.assert_array_equal(v, h.transpose(2, 0, 1))  # same field in both layouts (:62)


# ------------------------------------------------------------ golden fixtures
def test_setup_matches_reference_fixtures():
    np.testing.assert_array_equal(vertical_grid(4, 0.1), GOLD["grid_4_0.1"])
    np.testing.assert_array_equal(vertical_grid(128, 0.01), GOLD["grid_128_0.01"])
    for m in (1, 2, 4, 8, 13):
        for sphere in (True, False):
            tag = f"{'sphere' if sphere else 'planar'}_{m}"
            a, e, n, d = panel(m, sphere, 2.0)
            for got, key in ((a, "area"), (e, "east"), (n, "north"), (d, "diag")):
                np.testing.assert_array_equal(got.reshape(-1), GOLD[f"panel_{tag}_{key}"].reshape(-1))
    for n_z, h, om, la in ((2, 0.1, 1.0, 1.0), (16, 0.02, 6.71e-4, 3.32e-2), (64, 1e-2, 6.71e-4, 3.32e-2),
                           (12, 0.05, 0.3, 0.7)):
        tag = f"{n_z}_{h}_{om}_{la}"
        for got, key in zip(vertical_profile(vertical_grid(n_z, h), om, la), ("ap", "bp", "cp", "d")):
            np.testing.assert_array_equal(got, GOLD[f"prof_{tag}_{key}"])


@pytest.mark.parametrize("case", [(4, 8, True), (8, 16, True), (8, 16, False), (13, 7, True), (1, 12, True)])
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_operators_match_reference_fixtures(case, dt):
    m, n_z, sphere = case
    o = Oracle(Problem(m, n_z, sphere))
    tag = f"{m}_{n_z}_{'s' if sphere else 'p'}_{'f32' if dt == np.float32 else 'f64'}"
    x = o.random_field(5, dt)
    np.testing.assert_array_equal(x, GOLD[f"op_{tag}_x"])
    np.testing.assert_array_equal(o.apply(x), GOLD[f"op_{tag}_apply"])
    np.testing.assert_array_equal(o.precondition(x), GOLD[f"op_{tag}_prec"])
    u, p, q, z, r = (o.random_field(s, dt) for s in (101, 104, 105, 103, 102))
    u2, p2, q2, sg, _ = o.fused_spmv(u, p, q, z, 0.37, 0.21)
    for got, key in ((u2, "u"), (p2, "p"), (q2, "q")):
        np.testing.assert_array_equal(got, GOLD[f"op_{tag}_spmv_{key}"])
    assert sg == float(GOLD[f"op_{tag}_spmv_sigma"])
    r2, z2, rn, ka, _, _ = o.fused_prec(r, q, 0.37)
    np.testing.assert_array_equal(r2, GOLD[f"op_{tag}_prec2_r"])
    np.testing.assert_array_equal(z2, GOLD[f"op_{tag}_prec2_z"])
    assert [rn, ka] == list(GOLD[f"op_{tag}_prec2_rk"])
    assert [o.dot(u, p), o.nrm2(u), o.true_residual(u, r)] == list(GOLD[f"op_{tag}_dot"])


SOLVES = [
    ("s8_16_il", Problem(8, 16), np.float64, dict(epsilon=1e-8, maxiter=300, variant="interleaved")),
    ("s8_16_std", Problem(8, 16), np.float64, dict(epsilon=1e-8, maxiter=300, variant="standard")),
    ("s8_16_f32", Problem(8, 16), np.float32, dict(epsilon=1e-4, maxiter=200, variant="interleaved")),
    ("p4_8_std5", Problem(4, 8, False), np.float64, dict(epsilon=1e-300, maxiter=5, variant="standard")),
    ("s16_32_court", Problem(16, 32, True, 6.71e-4 * 16 ** 2), np.float64,
     dict(epsilon=1e-300, maxiter=50, variant="interleaved")),
    ("s1_16_il", Problem(1, 16), np.float64, dict(variant="interleaved")),
    ("s8_16_exh", Problem(8, 16), np.float64, dict(epsilon=1e-300, maxiter=3, variant="interleaved")),
]


@pytest.mark.parametrize("tag,prob,dt,kw", SOLVES, ids=[c[0] for c in SOLVES])
def test_solves_match_reference_fixtures(tag, prob, dt, kw):
    o = Oracle(prob)
    f = o.random_field(13 if tag.startswith("s1_") else 42, dt)
    u, res = o.solve(f, **kw)
    np.testing.assert_array_equal(u, GOLD[f"solve_{tag}_u"])
    np.testing.assert_array_equal(res.residual_history, GOLD[f"solve_{tag}_res"])
    np.testing.assert_array_equal(res.kappa_history, GOLD[f"solve_{tag}_kap"])
    np.testing.assert_array_equal(res.alpha_history, GOLD[f"solve_{tag}_alp"])
    np.testing.assert_array_equal(res.beta_history, GOLD[f"solve_{tag}_bet"])
    it, conv, tr = GOLD[f"solve_{tag}_meta"]
    assert (res.iterations, int(res.converged), res.true_residual) == (int(it), int(conv), tr)


def test_config1_matches_reference_fixture():
    """BASELINE config 1 (128x128x64 fp64, eps 1e-10): 88 iterations, bit-exact."""
    o = Oracle(Problem(128, 64))
    f = o.random_field(42)
    assert sha(f) == str(GOLD["c1_f_sha"])
    u, res = o.solve(f, epsilon=1e-10, maxiter=500)
    assert res.iterations == 88 == int(GOLD["c1_meta"][0])
    np.testing.assert_array_equal(res.residual_history, GOLD["c1_res"])
    np.testing.assert_array_equal(res.kappa_history, GOLD["c1_kap"])
    np.testing.assert_array_equal(res.alpha_history, GOLD["c1_alp"])
    np.testing.assert_array_equal(res.beta_history, GOLD["c1_bet"])
    assert sha(u) == str(GOLD["c1_u_sha"])
    assert res.true_residual == GOLD["c1_meta"][2]


def test_pairwise_sum_shape():
    """parallel.hpp:11-20: <= 8 sequential, else halves — independent of any worker split."""
    o = Oracle(Problem(2, 2))
    v = np.random.default_rng(0).standard_normal(1000)

    def ps(a):
        if len(a) <= 8:
            s = 0.0
            for x in a:
                s += x
            return s
        h = len(a) // 2
        return ps(a[:h]) + ps(a[h:])

    for n in (1, 7, 8, 9, 16, 17, 100, 1000):
        assert o.pairwise_sum(v[:n]) == ps(list(v[:n]))


# ------------------------------------------------------------ reference itself
@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("m,n_z,sphere", [(6, 10, True), (16, 9, False), (21, 5, True)])
def test_oracle_matches_reference_build(m, n_z, sphere):
    prob = Problem(m, n_z, sphere)
    o, r = Oracle(prob), Reference(prob, workers=3)
    for dt in (np.float64, np.float32):
        for layout in (0, 1):
            x = o.random_field(7, dt, layout)
            np.testing.assert_array_equal(x, r.random_field(7, dt, layout))
            np.testing.assert_array_equal(o.apply(x, layout), r.apply(x, layout))
            np.testing.assert_array_equal(o.precondition(x, layout), r.precondition(x, layout))
            f = o.random_field(42, dt, layout)
            for variant in ("standard", "interleaved"):
                uo, ro = o.solve(f, epsilon=1e-7, maxiter=200, variant=variant, layout=layout)
                ur, rr = r.solve(f, epsilon=1e-7, maxiter=200, variant=variant, layout=layout)
                np.testing.assert_array_equal(uo, ur)
                np.testing.assert_array_equal(ro.residual_history, rr.residual_history)
                assert ro.iterations == rr.iterations


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_reference_breakdown_and_flip():
    prob = Problem(4, 8)
    o, r = Oracle(prob).flip_d(), Reference(prob, flip_d=True)
    f = o.random_field(3)
    with pytest.raises(RuntimeError):
        o.solve(f, variant="standard")
    with pytest.raises(RuntimeError):
        r.solve(f, variant="standard")
