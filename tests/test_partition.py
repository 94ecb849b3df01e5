"""Partitioned (multi-rank) solve: BASELINE config 4's subtree split.

CPU (gloo, world_size 2): the partition map and each rank's layout agree
across ranks (every copy held exactly once, export slots consistent).
GPU (two ranks sharing one B200 over gloo -- this run has one GPU; NCCL
needs one device per rank): the assembled partitioned solve is bitwise equal
to the CPU oracle, iteration count included.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2501_08293_b200 import build, dopf, partition


@pytest.fixture(scope="module", autouse=True)
def _cuda_built():
    build.build_cuda()


def tiled_model(tiles=2):
    f = dopf.tiled_feeder("ieee8500", tiles, 850064)
    _, _, m = dopf.load_model(f, workers=4)
    m.precompute(4)
    return m


def test_partition_map_is_balanced_and_subtree_shaped():
    m = tiled_model(4)
    parts = partition.partition_subsystems(m, 4)
    assert parts.min() == 0 and parts.max() == 3
    ns = np.diff(m.z_offsets)
    rows = np.bincount(parts, weights=ns, minlength=4)
    assert rows.max() / rows.min() < 1.3
    # pieces of the walk are runs of whole tiles: a tile's subsystems sit on one rank
    tile_of = {}
    for s in range(m.S):
        cid = m.component_id(s)
        if "t0" in cid or "t1" in cid or "t2" in cid or "t3" in cid:
            key = cid.split("_")[0].split(":")[-1][-3:]
            tile_of.setdefault(key, set()).add(int(parts[s]))
    assert sum(len(v) for v in tile_of.values()) <= len(tile_of) + 3  # at most the cut tiles split


def test_part_layouts_cover_the_model():
    m = tiled_model(2)
    parts = partition.partition_subsystems(m, 3)
    infos = [partition.probe_part(m, 3, p, parts) for p in range(3)]
    assert sum(i["rows"] for i in infos) == m.total_local_vars
    assert len({i["max_export"] for i in infos}) == 1
    assert max(i["n_export"] for i in infos) == infos[0]["max_export"]
    assert sum(i["bytes_per_iteration"] for i in infos) > 0
    with pytest.raises(ValueError):
        partition.probe_part(m, 3, 3, parts)


WORKER = r"""
import os, sys, json
sys.path.insert(0, os.environ["REPO"])
import numpy as np, torch, torch.distributed as td
td.init_process_group("gloo")
rank, world = td.get_rank(), td.get_world_size()
from paper_2501_08293_b200 import dopf, partition
mode = os.environ["MODE"]
if mode.startswith("tiled"):
    f = dopf.tiled_feeder("ieee8500", int(mode[5:]), 850064)
else:
    f = dopf.synthetic_feeder(mode, int(os.environ["SEED"]))
_, _, m = dopf.load_model(f, workers=2)
m.precompute(2)
parts = partition.partition_subsystems(m, world)
infos = [None] * world
td.all_gather_object(infos, (partition.probe_part(m, world, rank, parts), parts.tolist()))
out = {"parts_equal": all(i[1] == infos[0][1] for i in infos),
       "rows": [i[0]["rows"] for i in infos], "max_export": [i[0]["max_export"] for i in infos],
       "n_export": [i[0]["n_export"] for i in infos], "N_z": m.total_local_vars}
if os.environ.get("SOLVE") == "1":
    torch.cuda.set_device(0)
    ps = partition.PartitionedSolver(0)
    ps.upload(m, parts)
    st = dopf.Settings(max_iter=int(os.environ["MAXIT"]))
    res = ps.assemble(ps.solve(st))
    if os.environ.get("REUPLOAD") == "1":  # pinned, same-structure re-upload: values-only fast path
        ps.solver.pin(m)
        ps.upload(m, parts)
        again = ps.assemble(ps.solve(st))
        out["reupload_same"] = bool(again.iterations == res.iterations and np.array_equal(again.x, res.x) and
                                    np.array_equal(again.z, res.z) and np.array_equal(again.lam, res.lam))
    if rank == 0:
        from oracle import oracle_py as O
        ref = O.solve(m, dopf.Settings(max_iter=int(os.environ["MAXIT"]), workers=4))
        out.update({"iterations": [res.iterations, ref.iterations], "status": [res.status, ref.status],
                    "x": bool(np.array_equal(res.x, ref.x)), "z": bool(np.array_equal(res.z, ref.z)),
                    "lam": bool(np.array_equal(res.lam, ref.lam)),
                    "obj": [res.objective, ref.objective],
                    "trace_rel": float(np.max(np.abs(res.trace[:, 1:] - ref.trace[:, 1:]) /
                                              np.maximum(1e-300, np.abs(ref.trace[:, 1:]))))})
if rank == 0:
    print("RESULT " + json.dumps(out))
td.destroy_process_group()
"""


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_ranks(tmp_path, world, env_extra, timeout=900):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, REPO=ROOT, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(script)]
    proc = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=timeout)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    line = [l for l in proc.stdout.splitlines() if l.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


def test_two_rank_partition_layouts_gloo(tmp_path):
    out = run_ranks(tmp_path, 2, {"MODE": "tiled2", "SOLVE": "0"})
    assert out["parts_equal"]
    assert sum(out["rows"]) == out["N_z"]
    assert out["max_export"][0] == out["max_export"][1] == max(out["n_export"])


@pytest.mark.gpu
@pytest.mark.parametrize("mode,world,maxit,reupload", [("tiled2", 2, 400, "1"), ("ieee123", 2, 50000, "0"),
                                                       ("tiled4", 3, 200, "0")])
def test_partitioned_solve_bitwise_two_ranks_one_gpu(tmp_path, mode, world, maxit, reupload):
    out = run_ranks(tmp_path, world, {"MODE": mode, "SEED": "123", "SOLVE": "1", "MAXIT": str(maxit),
                                      "REUPLOAD": reupload})
    if reupload == "1":
        assert out["reupload_same"], out
    assert out["iterations"][0] == out["iterations"][1]
    assert out["status"][0] == out["status"][1]
    assert out["x"] and out["z"] and out["lam"], out
    assert abs(out["obj"][0] - out["obj"][1]) <= 1e-6 * max(1.0, abs(out["obj"][1]))
    assert out["trace_rel"] <= 1e-9
