"""Partitioned solve under NCCL (graph-captured iterations) vs the oracle.

torchrun --nproc-per-node N tools/partition_nccl_check.py [mode] [max_iter]
(mode: ieee123 | tiledT). One GPU per rank; with one GPU use N = 1.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as td

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08293_b200 import dopf, partition  # noqa: E402

td.init_process_group("nccl")
rank, world = td.get_rank(), td.get_world_size()
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
mode = sys.argv[1] if len(sys.argv) > 1 else "ieee123"
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
f = dopf.tiled_feeder("ieee8500", int(mode[5:]), 850064) if mode.startswith("tiled") else \
    dopf.synthetic_feeder(mode, 123)
_, _, m = dopf.load_model(f, workers=4)
m.precompute(4)
ps = partition.PartitionedSolver(local)
ps.upload(m)
st = dopf.Settings(max_iter=maxit)
r1 = ps.assemble(ps.solve(st))
r2 = ps.assemble(ps.solve(st))  # graph replay path (captured on the first solve)
if rank == 0:
    from oracle import oracle_py as O
    ref = O.solve(m, dopf.Settings(max_iter=maxit, workers=8))
    for r in (r1, r2):
        print("iterations", r.iterations, ref.iterations, "bitwise",
              np.array_equal(r.x, ref.x) and np.array_equal(r.z, ref.z) and np.array_equal(r.lam, ref.lam))
td.destroy_process_group()
