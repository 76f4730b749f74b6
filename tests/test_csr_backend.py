"""backend = "csr" on the GPU: the reference's CsrBackend (solver.hpp:126-145)
as a drop-in — CSR matrix + stored tridiagonals assembled on the device,
driven by the standard PCG loop — bit-identical to the reference.

Golden fixtures: tests/golden/csr_golden.npz (tests/golden/make_csr_golden.py,
the unmodified reference's CsrBackend in oracle/_ref). The CSR summation
order follows the fields' layout, so the two layouts give (slightly)
different bits and both are checked. Also: the host assemble_csr (csr.hpp
drop-in) against the reference's own pybind module, p = 2 virtual slabs, the
configuration errors.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.oracle import Problem, Reference, ref_available

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = os.path.join(HERE, "golden", "csr_golden.npz")

CASES = {
    "s8_16": (Problem(8, 16), np.float64, dict(epsilon=1e-8, maxiter=300)),
    "p13_7": (Problem(13, 7, False), np.float64, dict(epsilon=1e-10, maxiter=300)),
    "s32_24_f32": (Problem(32, 24), np.float32, dict(epsilon=1e-4, maxiter=300)),
    "s64_32_fix": (Problem(64, 32), np.float64, dict(epsilon=1e-300, tau=1e-300, maxiter=25)),
}


def ctx_for(acg, prob, dtype=np.float64, slabs=1):
    g = acg.vertical_grid(prob.n_z, prob.h)
    pan = acg.cubed_sphere_panel(prob.m) if prob.sphere else acg.planar_panel(prob.m, prob.extent)
    cls = acg.OperatorContextF32 if dtype == np.float32 else acg.OperatorContext
    return cls(acg.vertical_profile(g, prob.omega2, prob.lambda2), pan, slabs=slabs)


def field(acg, prob, dt, layout):
    f = acg.random_field(prob.m, prob.n_z, 42, dtype="float32" if dt == np.float32 else "float64")
    return f if layout == 0 else np.ascontiguousarray(np.transpose(f, (1, 2, 0)))


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("case", sorted(CASES))
def test_csr_solve_bit_exact(acg, case, layout):
    prob, dt, kw = CASES[case]
    g = np.load(GOLD)
    key = f"{case}_L{layout}"
    ctx = ctx_for(acg, prob, dt)
    f = field(acg, prob, dt, layout)
    u, r = acg.solve(ctx, f, variant="standard", backend="csr",
                     layout="vertical" if layout == 0 else "horizontal", **kw)
    it, conv, tr = g[f"{key}_meta"]
    assert r.iterations == int(it) and r.converged == bool(conv)
    for k, name in (("res", "residual_history"), ("kap", "kappa_history"),
                    ("alp", "alpha_history"), ("bet", "beta_history")):
        assert np.array_equal(getattr(r, name), g[f"{key}_{k}"]), name
    assert r.true_residual == tr
    assert np.array_equal(u, g[f"{key}_u"])
    assert r.timings.setup_s > 0  # assembly counted as setup, like make_backend


def test_csr_device_arrays_and_slabs(acg):
    """CUDA arrays in/out, and p = 2 virtual slabs (ghost planes in the column
    indices), both against the reference's CsrBackend run live."""
    torch = pytest.importorskip("torch")
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    prob = Problem(64, 32)
    ref = Reference(prob)
    f = ref.random_field(42)
    uo, ro = ref.solve(f, variant="standard", backend="csr", epsilon=1e-10, maxiter=400)
    for slabs in (1, 2):
        ctx = ctx_for(acg, prob, slabs=slabs)
        u, r = acg.solve(ctx, torch.from_numpy(f).cuda(), variant="standard", backend="csr",
                         epsilon=1e-10, maxiter=400)
        assert r.iterations == ro.iterations
        assert np.array_equal(r.residual_history, ro.residual_history)
        assert np.array_equal(u.cpu().numpy(), uo)
        ctx.release_scratch()  # frees the assembled matrix too; a new solve re-assembles
        u2, r2 = acg.solve(ctx, f, variant="standard", backend="csr", epsilon=1e-10, maxiter=400)
        assert np.array_equal(u2, uo)


def test_csr_config_errors(acg):
    prob = Problem(4, 8)
    ctx = ctx_for(acg, prob)
    f = acg.random_field(4, 8, 1)
    with pytest.raises(ValueError, match="interleaved variant exists for the matrix-free"):
        acg.solve(ctx, f, variant="interleaved", backend="csr")
    with pytest.raises(ValueError):
        acg.solve(ctx, f, variant="standard", backend="dense")


def test_host_assemble_csr_matches_reference_module(acg):
    """csr.hpp's host assemble_csr == the reference's own module (oracle/_ref/anisocg,
    bindings.cpp:179-193), run in a subprocess (two pybind modules registering the
    same C++ type names cannot share a process)."""
    refmod = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(refmod, "anisocg")):
        pytest.skip("reference pybind module not built")
    cases = [(4, 8, True), (8, 16, False), (5, 3, True)]
    code = (
        "import sys, json, numpy as np\n"
        f"sys.path.insert(0, {refmod!r})\n"
        "import anisocg as a\n"
        "out = {}\n"
        f"for m, nz, sph in {cases!r}:\n"
        "    g = a.vertical_grid(nz, 0.01)\n"
        "    pan = a.cubed_sphere_panel(m) if sph else a.planar_panel(m, 2.0)\n"
        "    ctx = a.OperatorContext(a.vertical_profile(g, 6.71e-4, 3.32e-2), pan)\n"
        "    rp, ci, va = a.assemble_csr(ctx)\n"
        "    out[f'{m}_{nz}_{sph}'] = [rp.tolist(), ci.tolist(), [float(x).hex() for x in va]]\n"
        "print(json.dumps(out))\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    ref = json.loads(r.stdout)
    for m, nz, sph in cases:
        g = acg.vertical_grid(nz, 0.01)
        pan = acg.cubed_sphere_panel(m) if sph else acg.planar_panel(m, 2.0)
        ctx = acg.OperatorContext(acg.vertical_profile(g, 6.71e-4, 3.32e-2), pan)
        rp, ci, va = acg.assemble_csr(ctx)
        e_rp, e_ci, e_va = ref[f"{m}_{nz}_{sph}"]
        assert rp.tolist() == e_rp and ci.tolist() == e_ci
        assert [float(x).hex() for x in va] == e_va


def test_matrix_free_vs_csr_agree(acg):
    """test_solver.cpp:136-149: the two backends' standard-loop residual histories
    agree to 1e-13 * ||r0|| (different summation orders, same operator)."""
    prob = Problem(16, 32)
    ctx = ctx_for(acg, prob)
    f = acg.random_field(16, 32, 42)
    kw = dict(epsilon=1e-300, tau=1e-300, maxiter=50, variant="standard")
    _, rm = acg.solve(ctx, f, backend="matrix-free", **kw)
    _, rc = acg.solve(ctx, f, backend="csr", **kw)
    r0 = rm.residual_history[0]
    assert len(rm.residual_history) == len(rc.residual_history)
    assert np.abs(rm.residual_history - rc.residual_history).max() <= 1e-13 * r0


def test_csr_breakdown_message(acg):
    """A non-SPD operator (d negated, test_solver.cpp:194-204) on the CSR backend
    raises NumericalBreakdown with the reference's message where the reference's
    CsrBackend raises it (oracle/_ref run live)."""
    from oracle.oracle import Oracle
    from paper_1302_7193_b200 import capi
    prob = Problem(4, 8)
    o = Oracle(prob).flip_d()
    cctx = capi.Context(o.ap, o.bp, o.cp, o.d, o.area, o.east, o.north, o.diag)
    f = o.random_field(3)
    ff = cctx.field().upload(f)
    with pytest.raises(capi.BreakdownError) as ei:
        capi.solve(cctx, ff, variant=capi.STANDARD, backend=capi.CSR)
    if ref_available():
        with pytest.raises(RuntimeError) as er:
            Reference(prob, flip_d=True).solve(f, variant="standard", backend="csr")
        assert str(er.value).split(":")[0] in str(ei.value)
