"""Every kernel the library ships, not only the C3 defaults, is bit-exact.

Kernel choice is by shape and precision (no tuning switches since round 2):
K1 = k_thomas_tm (fp64, and fp32 with odd m) / k_thomas_tm2 (fp32, even m) /
k_thomas (z' in global memory: n_z*s > 1 KiB); K2 = k_fused_spmv_pair2 (fp64,
even m) / k_fused_spmv_quad (fp32, m % 4 == 0) / k_fused_spmv_pair (fp32, other
even m), k_fused_spmv_tile for odd m; reduction
stage 2 = k_tree2_wide / k_tree2_shfl / k_tree2 by leaf count. The worker
(tests/variant_worker.py) runs shapes that reach each of them, in one process
per launch-mode setting: the default, programmatic dependent launch off
(ACG_PDL=0), a reduction kernel after every sweep instead of the consumed
reductions of small single-slab grids (ACG_CONSUME=0), and narrow-panel K2
without the level split (ACG_KSPLIT=0).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = {
    "default": {},
    "no_pdl": {"ACG_PDL": "0"},
    "no_consume": {"ACG_CONSUME": "0"},
    "no_ksplit": {"ACG_KSPLIT": "0"},
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_bit_exact(name):
    env = dict(os.environ, OMP_NUM_THREADS="1", **VARIANTS[name])
    r = subprocess.run([sys.executable, os.path.join(HERE, "variant_worker.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "VARIANT_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
