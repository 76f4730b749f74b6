"""Multi-GPU runs on one node: one process per GPU, i-slabs.

Run when the box has at least N GPUs; skipped cleanly otherwise (this pool's
gpurun boxes have one GPU — the same code paths run with all ranks on one GPU
in tests/test_multirank_ipc.py and tests/test_bench_contract.py).

* peer-memory transport (CUDA IPC mailboxes over NVLink, release/acquire
  flags between devices) and NCCL transport (send/recv halos, all-gathered
  slab sums), N = 2, 4, 8: a solve bit-identical to the CPU reference
  (tests/mp_ipc_worker.py; slabs are reduction-tree nodes);
* bench.py --gpus N at C3 for both transports: the N-rank residual history
  equals the same iterations on one GPU bit for bit (verified_vs_1gpu).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def need(n):
    try:
        import torch
        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        have = 0
    if have < n:
        pytest.skip(f"needs {n} GPUs, this box has {have}")


@pytest.mark.parametrize("transport", ["ipc", "nccl"])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_ranks_on_separate_gpus_bit_exact(n, transport):
    need(n)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + 10 * n + (transport == "nccl")),
           os.path.join(HERE, "mp_ipc_worker.py"), "64", "24"]
    env = dict(os.environ, ACG_SAME_GPU="0", ACG_TEST_TRANSPORT=transport, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "IPC_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("transport", ["ipc", "nccl"])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_bench_scales_and_verifies(n, transport):
    need(n)
    env = dict(os.environ, OMP_NUM_THREADS="2")
    env.pop("ACG_SAME_GPU", None)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                        "--config", "c3", "--transport", transport, "--steps", "20", "--warmup", "3",
                        "--no-cpu", "--sustain-steps", "0"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip().startswith("{")][-1])
    assert d["n_gpus"] == n and d["value"] > 0
    v = d["verified_vs_1gpu"]
    assert v["ok"] is True and v["exact_tree"] is True


def test_nccl_communicator_single_rank(acg):
    """What the one-GPU pool can execute of the NCCL transport: ncclGetUniqueId,
    ncclCommInitRank and ncclCommDestroy through acg_comm_create/destroy, and a
    context placed on the communicator (one rank: its reduction needs no
    exchange) solving bit-identically to the CPU reference."""
    need(1)
    from oracle.oracle import Oracle, Problem
    from paper_1302_7193_b200 import capi
    o = Oracle(Problem(32, 16))
    comm = capi.Comm(0, 1, capi.Comm.unique_id(), 0)
    ctx = capi.Context(o.ap, o.bp, o.cp, o.d, o.area, o.east, o.north, o.diag, comm=comm)
    f = ctx.field().fill_random(42)
    u = ctx.field()
    r = capi.solve(ctx, f, u_out=u, epsilon=1e-9, maxiter=200)
    uo, ro = o.solve(o.random_field(42), epsilon=1e-9, maxiter=200)
    assert r["iterations"] == ro.iterations
    assert (r["residual_history"] == ro.residual_history).all()
    assert (u.download() == uo).all()
    for h in (f, u):
        h.close()
    ctx.close()
    comm.close()
