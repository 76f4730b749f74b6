"""Multi-process slab decomposition over the peer-memory transport
(acg_comm_create_ipc): 2 and 4 ranks, one process each, on GPU 0, solved
end to end and compared bit for bit with the CPU reference (mp_ipc_worker.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


# halo variants: fused into the sweeps (K1 puts the boundary planes into the
# neighbours' mailboxes, K2 acquires them; default) and copy + signal on a side
# stream overlapped with the interior sweep (ACG_FUSED_HALO=0; also the path of
# the standard loop and of odd m); odd m has no plane-range sweep, so its halo
# runs in stream order
HALO = {"fused": {}, "overlap": {"ACG_FUSED_HALO": "0"}}


@pytest.mark.parametrize("world,port,halo,m", [(2, 29611, "fused", 64), (4, 29612, "fused", 64),
                                               (2, 29613, "overlap", 64), (4, 29614, "overlap", 64),
                                               (2, 29615, "fused", 66),
                                               (2, 29622, "fused", 65),
                                               # two planes per rank; one plane per rank
                                               # (4-column slabs are not tree nodes:
                                               # compared within the fp64 tolerances)
                                               (4, 29616, "fused", 8), (4, 29617, "fused", 4),
                                               # fp32: k_thomas_tm2 puts, k_fused_spmv_pair reads
                                               (2, 29618, "fused-f32", 64),
                                               (4, 29619, "fused-f32", 64),
                                               (2, 29620, "overlap-f32", 64)])
def test_ipc_ranks_bit_exact(world, port, halo, m):
    f32 = halo.endswith("-f32")
    halo = halo[:-4] if f32 else halo
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(HERE, "mp_ipc_worker.py"), str(m), "24"] + (["f32"] if f32 else [])
    env = dict(os.environ, ACG_SAME_GPU="1", OMP_NUM_THREADS="1", **HALO[halo])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "IPC_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
