"""Probe: can two ranks share one GPU in an NCCL communicator (acg_comm)?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_1302_7193_b200 import capi

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
obj = [capi.Comm.unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
try:
    comm = capi.Comm(rank, world, obj[0], 0)
    print(f"rank {rank}: comm ok", flush=True)
except Exception as e:
    print(f"rank {rank}: comm failed: {e}", flush=True)
dist.destroy_process_group()
