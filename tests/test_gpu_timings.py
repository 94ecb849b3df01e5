"""PhaseTimings of the device solves (reference admm.hpp:104-106, measured at
admm.cpp:182-217 and reported by the CLI, tools/main.cpp:140-143): the loop's
device time split into global / local / dual by the kernels' own clocks
(resident: block 0's phase clock every 32nd iteration; streaming: kernel
%globaltimer stamps). Each share is positive where the phase is separate and
the split adds up to the measured loop time."""
import json
import subprocess

import pytest

from conftest import fixture_path
from paper_2501_08293_b200 import build, dopf, partition

pytestmark = pytest.mark.gpu


def check_split(res, dual_separate=True):
    t = res.timings
    assert t["global"] > 0 and t["local"] > 0, t
    if dual_separate:
        assert t["dual"] > 0, t
    else:
        assert t["dual"] == 0.0, t
    total = t["global"] + t["local"] + t["dual"]
    assert abs(total - t["solve"]) <= 1e-9 + 1e-6 * t["solve"], t
    # the GEMV dominates the local share on these feeders
    assert t["local"] > 0.1 * t["solve"], t


@pytest.mark.parametrize("path", ["resident", "stream"])
def test_solve_phase_timings(path):
    f = dopf.synthetic_feeder("ieee123", 123)
    _, _, m = dopf.load_model(f, workers=4)
    m.precompute(4)
    s = dopf.CudaSolver(0)
    s.set_path(path)
    s.upload(m)
    res = s.solve(dopf.Settings(max_iter=500))
    check_split(res, dual_separate=path == "resident")


def test_batch_phase_timings():
    from paper_2501_08293_b200 import scenarios
    from paper_2501_08293_b200.batch import BatchSolver
    bs = BatchSolver(0)
    bs.upload(scenarios.build_scenarios("ieee13", 13, range(3)))
    for res in bs.solve(dopf.Settings(max_iter=300)):
        check_split(res)


def test_partitioned_phase_timings():
    f = dopf.synthetic_feeder("ieee123", 123)
    _, _, m = dopf.load_model(f, workers=4)
    m.precompute(4)
    ps = partition.NcclPartitionedSolver(0, 1, 0, partition.nccl_unique_id())
    ps.upload(m)
    res = ps.solve(dopf.Settings(max_iter=500))
    check_split(res, dual_separate=False)


def test_cli_report_has_device_phase_timings(tmp_path):
    rep = tmp_path / "r.json"
    p = subprocess.run([build.CLI, "solve", "--input", fixture_path("four_bus_delta"), "--eps-rel", "1e-4",
                        "--report", str(rep)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    t = json.loads(rep.read_text())["timings_sec"]
    assert t["global"] > 0 and t["local"] > 0 and t["dual"] > 0 and t["precompute"] > 0, t
