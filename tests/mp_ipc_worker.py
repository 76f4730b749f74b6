"""Worker for tests/test_multirank_ipc.py (run under torch.distributed.run).

Each rank owns one i-slab of the context; the slabs talk through the peer-memory
transport (acg_comm_create_ipc: CUDA IPC mailboxes, release/acquire flags), all
ranks on GPU 0 here (the same code maps peer GPUs over NVLink on a multi-GPU
node). Rank 0 gathers the slabs and checks them bit for bit against the CPU
reference restatement (tree-aligned slabs reproduce the reference's reduction
order exactly).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle.oracle import Oracle, Problem  # noqa: E402
from paper_1302_7193_b200 import capi  # noqa: E402


def main():
    m, n_z = int(sys.argv[1]), int(sys.argv[2])
    f32 = len(sys.argv) > 3 and sys.argv[3] == "f32"
    npdt = np.float32 if f32 else np.float64
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = 0 if os.environ.get("ACG_SAME_GPU", "1") == "1" else int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    if os.environ.get("ACG_TEST_TRANSPORT") == "nccl":  # one GPU per rank (NCCL refuses shared GPUs)
        uid = [capi.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = capi.Comm(rank, world, uid[0], dev)
    else:
        uid = [os.urandom(16) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = capi.Comm.ipc(rank, world, uid[0], dev)
    o = Oracle(Problem(m, n_z))
    ctx = capi.Context(o.ap, o.bp, o.cp, o.d, o.area, o.east, o.north, o.diag, device=dev,
                       comm=comm, dtype=capi.F32 if f32 else capi.F64)
    info = ctx.info()
    f = ctx.field().fill_random(42)
    u = ctx.field()
    res = capi.solve(ctx, f, u_out=u, epsilon=1e-9 if not f32 else 1e-4, maxiter=400)
    x = o.random_field(7, dtype=npdt)
    fx, fy = ctx.field().upload(x), ctx.field()
    capi.apply(ctx, fx, fy)
    tr = capi.true_residual(ctx, u, f)
    parts = [None] * world
    dist.gather_object((info["i_begin"], u.download(scope=capi.HOST_LOCAL),
                        fy.download(scope=capi.HOST_LOCAL)), parts if rank == 0 else None, dst=0)
    if rank == 0:
        parts.sort(key=lambda t: t[0])
        ug = np.concatenate([p_[1] for p_ in parts], axis=0)
        yg = np.concatenate([p_[2] for p_ in parts], axis=0)
        uo, ro = o.solve(o.random_field(42, dtype=npdt), epsilon=1e-9 if not f32 else 1e-4,
                         maxiter=400)
        if info["exact_tree"]:  # slabs are nodes of the reference's tree: bit for bit
            ok = (res["iterations"] == ro.iterations
                  and np.array_equal(res["residual_history"], ro.residual_history)
                  and np.array_equal(res["kappa_history"], ro.kappa_history)
                  and np.array_equal(ug, uo) and np.array_equal(yg, o.apply(x))
                  and res["true_residual"] == ro.true_residual and tr == ro.true_residual)
        else:  # slab sums combined pairwise: the north-star tolerances
            tol = 1e-4 if f32 else 1e-10
            n = min(len(res["residual_history"]), len(ro.residual_history))
            r0 = ro.residual_history[0]
            ok = (abs(res["iterations"] - ro.iterations) <= 1
                  and np.max(np.abs(np.asarray(res["residual_history"][:n])
                                    - ro.residual_history[:n])) <= tol * r0
                  and np.max(np.abs(ug - uo)) <= tol * np.max(np.abs(uo))
                  and np.array_equal(yg, o.apply(x)))
        print(f"world={world} iterations={res['iterations']} (ref {ro.iterations}) "
              f"exact_tree={info['exact_tree']} {'IPC_OK' if ok else 'IPC_MISMATCH'}", flush=True)
    dist.barrier()
    for fl in (f, u, fx, fy):
        fl.close()
    ctx.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
