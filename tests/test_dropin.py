"""The reference's Python boundary, unchanged, on the B200 library.

oracle/Makefile compiles the reference's own proj/python/bindings.cpp,
UNMODIFIED, against this repo's drop-in headers (include/anisocg/*.hpp,
including csr.hpp) and links it to libacg_cuda.so (oracle/_ref/dropin/). Next to
it sit byte-for-byte copies of the reference's python/anisocg/__init__.py and
tests/python/test_smoke.py (sha256 pinned below). The reference's 11 smoke
tests then run verbatim twice:

  * against that module (the reference's binding code over the B200 kernels);
  * against this repo's own ``anisocg`` package (paper_1302_7193_b200/_anisocg).

On a machine without a GPU only the host-only tests are run (setup and cost
tables); compute calls must fail loudly there, never fall back.

The same holds one level down: the reference's own C++ unit tests
(proj/tests/test_{field,grid,profile,operator,solver,cost_model}.cpp with
its oracles.hpp), compiled UNMODIFIED against include/anisocg/*.hpp and linked
to libacg_cuda.so (oracle/_ref/cpptests/, with tests/refcpp/doctest.h standing
in for the absent doctest header), must pass all 59 test cases on the GPU.
"""
import hashlib
import os
import subprocess
import sys

import pytest

from conftest import gpu_available

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin")
SMOKE = os.path.join(ROOT, "oracle", "_ref", "smoke")
# proj/tests/python/test_smoke.py and proj/python/anisocg/__init__.py of the reference
SMOKE_SHA = "59c65009605134a42cabf03b9620356f823b5ca0a3da05ea55792f3d0ad5ad42"
INIT_SHA = "1529dc14e5e577c6650ae9bf103e3a8c0d52c067fec1d9ce7cbc68dcb684abfe"
HOST_ONLY = "grading or partition or cost_model"


def sha(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def built():
    if not os.path.isdir(os.path.join(DROPIN, "anisocg")):
        pytest.skip("oracle/_ref/dropin not built (needs /root/reference at build time)")


def run_smoke(where, pythonpath, select=None):
    env = dict(os.environ, PYTHONPATH=pythonpath, OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "test_smoke.py"]
    if select:
        cmd += ["-k", select]
    return subprocess.run(cmd, cwd=where, env=env, capture_output=True, text=True, timeout=600)


def test_copies_are_verbatim():
    built()
    assert sha(os.path.join(DROPIN, "test_smoke.py")) == SMOKE_SHA
    assert sha(os.path.join(SMOKE, "test_smoke.py")) == SMOKE_SHA
    assert sha(os.path.join(DROPIN, "anisocg", "__init__.py")) == INIT_SHA
    ref = "/root/reference/proj/tests/python/test_smoke.py"
    if os.path.exists(ref):
        assert sha(ref) == SMOKE_SHA


def test_reference_binding_links_the_b200_library():
    built()
    so = [f for f in os.listdir(os.path.join(DROPIN, "anisocg")) if f.startswith("_anisocg")]
    assert so
    out = subprocess.run(["ldd", os.path.join(DROPIN, "anisocg", so[0])], capture_output=True,
                         text=True).stdout
    line = [l for l in out.splitlines() if "libacg_cuda.so" in l]
    assert line and "not found" not in line[0], out


@pytest.mark.skipif(gpu_available(), reason="the GPU run executes the whole file")
def test_reference_smoke_host_only_subset():
    built()
    for where, path in ((DROPIN, DROPIN), (SMOKE, ROOT)):
        r = run_smoke(where, path, HOST_ONLY)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
        assert "3 passed" in r.stdout, r.stdout[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("module", ["reference-binding", "repo-package"])
def test_reference_smoke_all_eleven(module):
    built()
    where, path = (DROPIN, DROPIN) if module == "reference-binding" else (SMOKE, ROOT)
    r = run_smoke(where, path)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "11 passed" in r.stdout, r.stdout[-2000:]


CPPTESTS = os.path.join(ROOT, "oracle", "_ref", "cpptests", "ref_unit_tests")


@pytest.mark.gpu
def test_reference_cpp_unit_tests_all_pass():
    if not os.path.exists(CPPTESTS):
        pytest.skip("oracle/_ref/cpptests not built (needs /root/reference at build time)")
    r = subprocess.run([CPPTESTS], capture_output=True, text=True, timeout=900, cwd=ROOT)
    summary = [l for l in r.stdout.splitlines() if l.startswith("[refcpp]")]
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert summary and "| 59 passed | 0 failed |" in summary[-1], r.stdout[-3000:]
    assert summary[-1].rstrip().endswith("| 0 failed"), summary[-1]
