"""Every shipped kernel variant, not only the defaults, is bit-exact.

The defaults are K1 = k_thomas_tm (fp64) / k_thomas_tm2 (fp32), K2 =
k_fused_spmv_pair2 (fp64) / k_fused_spmv_pair (fp32), stage 2 = k_tree2_wide,
programmatic dependent launch on. The ACG_* switches below select the other
kernels the library ships (fallbacks, experiments kept for A/B runs); each runs
in its own process (tests/variant_worker.py) against the CPU oracle.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = {
    "thomas_legacy": {"ACG_THOMAS_TM": "0"},            # k_thomas (global-memory z')
    "thomas_legacy_w2": {"ACG_THOMAS_TM": "0", "ACG_THOMAS": "2,4,7"},
    "thomas_tm_fp32": {"ACG_THOMAS_TM2": "0"},          # one column per thread for fp32 too
    "thomas_tm2_fp64": {"ACG_THOMAS_TM2": "1"},         # two columns per thread for fp64 too
    "thomas_tma": {"ACG_THOMAS_TMA": "1"},              # TMA-fed tiles
    "thomas_cp8": {"ACG_THOMAS_TM": "8,15,15"},
    "thomas_q1": {"ACG_THOMAS_TM": "q1"},
    "thomas_x1": {"ACG_THOMAS_TM": "4,15,15,1"},        # four planes x 32 j per CTA
    "thomas_tpc3": {"ACG_TM_TPC": "3"},                 # three planes per CTA
    "spmv_plain": {"ACG_SPMV": "plain"},
    "spmv_ring": {"ACG_SPMV": "ring"},
    "spmv_tile": {"ACG_SPMV": "tile"},
    "spmv_pair": {"ACG_SPMV": "pair"},
    "spmv_pair2": {"ACG_SPMV": "pair2"},
    "tree2_shfl": {"ACG_TREE2": "shfl"},
    "tree2_legacy": {"ACG_TREE2": "legacy"},
    "no_fused_reduce": {"ACG_FUSED_REDUCE": "0"},       # per-column partials + k_tree1
    "cta_finish": {"ACG_CTA_FINISH": "1"},              # last CTA finishes the reduction
    "no_pdl": {"ACG_PDL": "0"},
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_bit_exact(name):
    env = dict(os.environ, OMP_NUM_THREADS="1", **VARIANTS[name])
    r = subprocess.run([sys.executable, os.path.join(HERE, "variant_worker.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "VARIANT_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
