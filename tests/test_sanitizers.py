"""compute-sanitizer over the kernels (racecheck / synccheck /
memcheck on small grids; the reference guards races by construction,
operator.hpp:158, :293, and checks determinism, test_solver.cpp:178-192).

The kernels carry hand-rolled cp.async rings, TMEM allocation, programmatic
dependent launches and, across ranks, release/acquire flags in peer memory.
Each tool runs tests/sanitize_worker.py (single process: every kernel family,
fp64/fp32, exact/fast, 1 and 2 slabs, parity-checked) and a 2-rank
peer-memory solve (tests/mp_ipc_worker.py, each rank under the sanitizer);
all must report zero errors. The logs are kept under gpurun_out/ when that
directory exists (tests/../gpurun_out).
"""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
TOOLS = ["memcheck", "racecheck", "synccheck", "initcheck"]


def sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    return exe


def keep_log(name, text):
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, f"sanitizer_{name}.log"), "w") as fh:
            fh.write(text)


@pytest.mark.parametrize("tool", TOOLS)
def test_single_process_clean(tool):
    cmd = [sanitizer(), "--tool", tool, "--error-exitcode", "97", "--print-limit", "50",
           sys.executable, os.path.join(HERE, "sanitize_worker.py")]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    log = r.stdout + r.stderr
    keep_log(tool, log)
    assert r.returncode == 0, log[-4000:]
    assert "SANITIZE_DONE" in r.stdout, log[-4000:]
    assert "ERROR SUMMARY: 0 errors" in log, log[-4000:]


@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_two_rank_peer_memory_clean(tool):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29640 + TOOLS.index(tool)),
           "--no-python", sanitizer(), "--tool", tool, "--error-exitcode", "97",
           sys.executable, os.path.join(HERE, "mp_ipc_worker.py"), "64", "24"]
    env = dict(os.environ, ACG_SAME_GPU="1", OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    log = r.stdout + r.stderr
    keep_log(f"ipc_{tool}", log)
    assert r.returncode == 0, log[-4000:]
    assert "IPC_OK" in r.stdout, log[-4000:]
    assert log.count("ERROR SUMMARY: 0 errors") == 2, log[-4000:]
