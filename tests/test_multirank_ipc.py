"""Multi-process slab decomposition over the peer-memory transport
(acg_comm_create_ipc): 2 and 4 ranks, one process each, on GPU 0, solved
end to end and compared bit for bit with the CPU reference (mp_ipc_worker.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("world,port", [(2, 29611), (4, 29612)])
def test_ipc_ranks_bit_exact(world, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(HERE, "mp_ipc_worker.py"), "64", "24"]
    env = dict(os.environ, ACG_SAME_GPU="1", OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "IPC_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
