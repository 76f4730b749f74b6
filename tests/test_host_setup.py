"""The product's host-side setup (paper_1302_7193_b200/csrc/host/*.cpp through
_anisocg) and the C ABI library, checked on CPU (no GPU needed).

Setup coefficients must be bit-identical to the reference's: every later
comparison (GPU vs CPU) starts from them.
"""
import math
import os
import re

import numpy as np
import pytest

from conftest import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))


def test_setup_bit_identical_to_reference(acg):
    np.testing.assert_array_equal(acg.vertical_grid(4, 0.1).r, GOLD["grid_4_0.1"])
    np.testing.assert_array_equal(acg.vertical_grid(128, 0.01).r, GOLD["grid_128_0.01"])
    for m in (1, 2, 4, 8, 13):
        for sphere in (True, False):
            g = acg.cubed_sphere_panel(m) if sphere else acg.planar_panel(m, 2.0)
            tag = f"{'sphere' if sphere else 'planar'}_{m}"
            for got, key in ((g.cell_area, "area"), (g.alpha_east, "east"), (g.alpha_north, "north"),
                             (g.alpha_diag, "diag")):
                np.testing.assert_array_equal(got.reshape(-1), GOLD[f"panel_{tag}_{key}"].reshape(-1))
    for n_z, h, om, la in ((2, 0.1, 1.0, 1.0), (16, 0.02, 6.71e-4, 3.32e-2), (64, 1e-2, 6.71e-4, 3.32e-2),
                           (12, 0.05, 0.3, 0.7)):
        p = acg.vertical_profile(acg.vertical_grid(n_z, h), om, la)
        tag = f"{n_z}_{h}_{om}_{la}"
        for got, key in ((p.a_prime, "ap"), (p.b_prime, "bp"), (p.c_prime, "cp"), (p.d, "d")):
            np.testing.assert_array_equal(got, GOLD[f"prof_{tag}_{key}"])


def test_reference_smoke_surface(acg):
    """The host-only checks of proj/tests/python/test_smoke.py, through `import anisocg`."""
    import anisocg
    grid = anisocg.vertical_grid(4, 0.1)
    np.testing.assert_allclose(grid.r, [1.0, 1.00625, 1.025, 1.05625, 1.1], rtol=1e-15)
    assert grid.r[0] == 1.0 and grid.r[-1] == 1.1
    pan = anisocg.cubed_sphere_panel(8)
    assert pan.cell_area.shape == (8, 8) and abs(pan.cell_area.sum() - 4 * math.pi / 6) < 1e-12
    np.testing.assert_allclose(anisocg.planar_panel(3, 3.0).alpha_diag, [[2, 3, 2], [3, 4, 3], [2, 3, 2]])
    prof = anisocg.vertical_profile(anisocg.vertical_grid(8, 0.01), 0.5, 0.25)
    np.testing.assert_allclose(prof.a_prime, -1.0 / 0.5, rtol=1e-14)
    assert prof.c_prime[0] == 0.0 and prof.b_prime[-1] == 0.0
    assert anisocg.cost_model("pcg_total", "none") == (46, 40)
    assert anisocg.cost_model("interleaved_total", "columns_cached") == (47, 20)
    with pytest.raises(ValueError):
        anisocg.cost_model("bogus", "none")
    g2 = anisocg.anisotropy(anisocg.planar_panel(4, 2.0), anisocg.vertical_grid(8, 0.01), 3.32e-2)
    assert g2.shape == (4, 4, 8) and g2.min() > 1.0
    with pytest.raises(ValueError):
        anisocg.vertical_grid(0, 0.1)
    with pytest.raises(ValueError):
        anisocg.planar_panel(4, 0.0)
    with pytest.raises(ValueError):
        anisocg.vertical_profile(anisocg.vertical_grid(4, 0.1), 0.0, 1.0)


def test_c_abi_exports_every_declared_symbol():
    from paper_1302_7193_b200 import capi
    header = open(os.path.join(ROOT, "include", "acg.h")).read()
    declared = set(re.findall(r"\b(acg_[a-z0-9_]+)\s*\(", header))
    assert len(declared) > 40
    import ctypes
    lib = ctypes.CDLL(capi.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert capi.lib().acg_abi_version() == 2


def test_partition_plan_is_tree_aligned():
    """Slabs are nodes of the reference's pairwise tree when p = 2^k divides m."""
    from paper_1302_7193_b200 import capi
    assert capi.partition_plan(1024, 8) == ([0, 128, 256, 384, 512, 640, 768, 896, 1024], True)
    assert capi.partition_plan(64, 4) == ([0, 16, 32, 48, 64], True)
    ib, ex = capi.partition_plan(40, 3)
    assert ib[0] == 0 and ib[-1] == 40 and not ex
    assert capi.partition_plan(96, 1) == ([0, 96], True)
    with pytest.raises(ValueError):
        capi.partition_plan(4, 8)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu(acg):
    """No CPU fallback: compute entry points raise when no CUDA device exists."""
    g = acg.vertical_grid(4, 0.01)
    with pytest.raises(RuntimeError):
        acg.OperatorContext(acg.vertical_profile(g, 6.71e-4, 3.32e-2), acg.cubed_sphere_panel(2))
    with pytest.raises(RuntimeError):
        acg.random_field(2, 4, 1)


def test_parallel_hpp_pairwise_sum_matches_the_oracle(tmp_path):
    """include/anisocg/parallel.hpp (host pairwise_sum, parallel.hpp:11-20 of the
    reference) sums in the same fixed tree as the oracle's restatement."""
    import shutil
    import subprocess
    from oracle.oracle import Oracle, Problem
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not installed")
    src = tmp_path / "ps.cpp"
    src.write_text(
        '#include <cstdio>\n#include <vector>\n#include "anisocg/parallel.hpp"\n'
        "int main() { std::size_t n; std::vector<double> v;\n"
        '  while (std::scanf("%zu", &n) == 1) { v.resize(n);\n'
        '    for (auto& x : v) std::scanf("%la", &x);\n'
        '    std::printf("%a\\n", anisocg::pairwise_sum(v.data(), v.size())); } }\n')
    exe = tmp_path / "ps"
    subprocess.run([gxx, "-O2", "-std=c++20", "-ffp-contract=off", "-I",
                    os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    rng = np.random.default_rng(7)
    sizes = [0, 1, 7, 8, 9, 16, 17, 100, 1023, 4096, 65537]
    arrays = [rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8, n) for n in sizes]
    inp = "".join(f"{a.size}\n" + "".join(f"{float(x).hex()}\n" for x in a) for a in arrays)
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True)
    got = [float.fromhex(l) for l in out.stdout.split()]
    o = Oracle(Problem(4, 2))
    want = [o.pairwise_sum(a) if a.size else 0.0 for a in arrays]
    assert got == want
