"""Multi-process i-slab decomposition on CPU (torch.distributed gloo, world 2 and 4).

Each rank owns the slab libacg_cuda.so's own partition plan assigns it
(acg_partition_plan), exchanges ghost planes with its neighbours, all-gathers
the slab sums of its reductions and replicates the scalar recurrences — the
host logic of the multi-GPU path (acg_runtime.cu halo()/reduce()), restated in
numpy by tests/slab_sim.py. The decomposed solve must equal the full-domain
oracle bit for bit when the plan is tree-aligned, and to 1e-13*||r0||
otherwise.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n_z, maxiter, eps, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle, Problem
    from paper_1302_7193_b200 import capi
    from slab_sim import Slab

    o = Oracle(Problem(m, n_z))
    ib, exact = capi.partition_plan(m, world)
    f = o.random_field(42)
    slab = Slab(o, ib[rank], ib[rank + 1], rank, world, exact)
    u, hist, it = slab.solve(f, eps, 1e-20, maxiter)
    parts = [None] * world
    dist.all_gather_object(parts, u)
    if rank == 0:
        np.savez(os.path.join(out_dir, f"res_{world}.npz"), u=np.concatenate(parts, axis=0),
                 hist=np.array(hist), it=it, exact=exact)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n_z", [(2, 16, 12), (4, 16, 12), (2, 12, 8), (3, 12, 8)])
def test_slab_solve_matches_full_domain(tmp_path, world, m, n_z):
    from oracle.oracle import Oracle, Problem
    from paper_1302_7193_b200 import capi

    eps, maxiter = 1e-9, 300
    mp.start_processes(_worker, args=(world, _free_port(), m, n_z, maxiter, eps, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    res = np.load(tmp_path / f"res_{world}.npz")
    o = Oracle(Problem(m, n_z))
    uo, ro = o.solve(o.random_field(42), epsilon=eps, maxiter=maxiter)
    _, exact = capi.partition_plan(m, world)
    assert bool(res["exact"]) == exact
    if exact:
        assert int(res["it"]) == ro.iterations
        np.testing.assert_array_equal(res["hist"], ro.residual_history)
        np.testing.assert_array_equal(res["u"], uo)
    else:
        assert abs(int(res["it"]) - ro.iterations) <= 1
        n = min(len(res["hist"]), len(ro.residual_history))
        r0 = ro.residual_history[0]
        assert np.abs(res["hist"][:n] - ro.residual_history[:n]).max() <= 1e-13 * r0
