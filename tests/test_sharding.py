"""Multi-rank host logic on CPU (gloo, world_size 2): the scenario sharding
rule (reference parallel.cpp:7-21) and the bench's max-over-ranks timing
reduction, run exactly as torchrun would launch them."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT
from paper_2501_08293_b200 import scenarios


def test_shard_rule_matches_reference():
    # parallel.cpp:7-21: contiguous, balanced, first (count % parts) one longer
    assert [scenarios.shard(10, 3, i) for i in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert [scenarios.shard(2, 4, i) for i in range(4)] == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for count in (0, 1, 7, 4096):
        for parts in (1, 2, 3, 8):
            r = [scenarios.shard(count, parts, i) for i in range(parts)]
            assert r[0][0] == 0 and r[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [e - b for b, e in r]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        scenarios.shard(4, 2, 2)


WORKER = r"""
import os, sys, json
sys.path.insert(0, os.environ["REPO"])
import torch, torch.distributed as td
from paper_2501_08293_b200 import scenarios
td.init_process_group("gloo")
rank, world = td.get_rank(), td.get_world_size()
b, e = scenarios.shard(int(os.environ["COUNT"]), world, rank)
models = scenarios.build_scenarios("ieee13", 13, range(b, e), 2)
mine = [m.total_local_vars for m in models]
allv = [None] * world
td.all_gather_object(allv, (rank, b, e, mine))
t = torch.tensor([float(rank + 1), float(len(mine))], dtype=torch.float64)
ts = [torch.zeros_like(t) for _ in range(world)]
td.all_gather(ts, t)
if rank == 0:
    print(json.dumps({"shards": allv, "max_t": max(float(x[0]) for x in ts),
                      "total": sum(float(x[1]) for x in ts)}))
td.destroy_process_group()
"""


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_scenario_sharding_gloo(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, REPO=ROOT, COUNT="5")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(script)]
    proc = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=300)
    assert proc.returncode == 0, proc.stderr[-2000:]
    import json
    line = [l for l in proc.stdout.splitlines() if l.startswith("{")][-1]
    out = json.loads(line)
    shards = sorted(out["shards"])
    assert [(s[1], s[2]) for s in shards] == [(0, 3), (3, 5)]
    assert out["total"] == 5 and out["max_t"] == 2.0
    assert all(v == shards[0][3][0] for s in shards for v in s[3])  # same structure per scenario
