"""Report and wire formats (io.hpp): the B200 build's writers against the
reference's own io.cpp compiled from source (oracle/_ref/libanisocg_io_ref.so),
byte for byte. CPU only (no GPU call)."""
import ctypes as C
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFIO = os.path.join(ROOT, "oracle", "_ref", "libanisocg_io_ref.so")


@pytest.fixture(scope="module")
def refio():
    if not os.path.exists(REFIO):
        pytest.skip("reference io harness not built (oracle/Makefile)")
    lib = C.CDLL(REFIO)
    for name in ("ref_residual_csv", "ref_cost_model_csv", "ref_geometry_csv", "ref_dump_field"):
        getattr(lib, name).restype = C.c_long
    return lib


def _call(fn, *args):
    n = fn(*args, None, 0)
    buf = C.create_string_buffer(n)
    fn(*args, buf, n)
    return buf.raw[:n]


@pytest.fixture(scope="module")
def report():
    from paper_1302_7193_b200 import report as r
    return r


def test_residual_csv(refio, report):
    rng = np.random.default_rng(3)
    for h in (np.array([2.5]), np.abs(rng.standard_normal(40)) * 10.0 ** -rng.integers(0, 12, 40),
              np.array([0.0, 0.0]), np.array([])):
        h = np.ascontiguousarray(h, dtype=np.float64)
        want = _call(refio.ref_residual_csv, h.ctypes.data_as(C.c_void_p), len(h))
        assert report.residual_csv(h).encode() == want


def test_cost_model_csv(refio, report):
    assert report.cost_model_csv().encode() == _call(refio.ref_cost_model_csv)


@pytest.mark.parametrize("m,sphere", [(1, True), (4, True), (7, False), (16, True)])
def test_geometry_csv(refio, report, m, sphere):
    import paper_1302_7193_b200 as acg
    g = acg.cubed_sphere_panel(m) if sphere else acg.planar_panel(m, 2.0)
    want = _call(refio.ref_geometry_csv, m, 1 if sphere else 0, C.c_double(2.0))
    assert report.geometry_csv(g).encode() == want


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("layout", ["vertical", "horizontal"])
def test_dump_field(refio, report, dtype, layout):
    m, nz = 5, 3
    shape = (m, m, nz) if layout == "vertical" else (m, nz, m)
    x = np.random.default_rng(1).standard_normal(shape).astype(dtype)
    want = _call(refio.ref_dump_field, m, nz, 1 if layout == "horizontal" else 0,
                 1 if dtype == np.float32 else 0, x.ctypes.data_as(C.c_void_p))
    assert report.dump_field(x, layout=layout) == want


def test_solve_json_and_bench_row(report):
    from types import SimpleNamespace
    t = SimpleNamespace(spmv=0.0, prec=0.0, blas=0.0, fused_spmv=0.5, fused_prec=0.25,
                        setup=0.125, total=1.0)
    res = SimpleNamespace(iterations=3, converged=False, true_residual=0.5,
                          residual_history=[4.0, 2.0, 1.0, 0.5], timings=t)
    j = report.solve_json(res, m=8, nz=4, h_atmos=0.01, omega2=6.71e-4, lambda2=3.32e-2)
    assert j["residual0"] == 4.0 and j["rel_residual"] == 0.125 and j["rhs"] == "splitmix64-uniform"
    assert j["timings"]["fused_spmv_s"] == 0.5 and "extent" not in j
    row = report.bench_csv_row(res, iters=100, m=8, nz=4)
    assert len(row.split(",")) == len(report.BENCH_CSV_HEADER.split(","))
    assert row.startswith("matrix-free,interleaved,vertical,double,1,8,4,100,125,8.75,")
