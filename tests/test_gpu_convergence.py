"""Parity to convergence on the two large BASELINE configs.

north_star: "identical iteration count to convergence" on every named config
(reference acceptance criteria, proj/tests/acceptance.cpp:89-134; termination
fidelity :255-306). The bench solves these exact inputs, so they are
compared with the oracle (the restated admm.cpp:172-244) end to end:

- configs[3]: the 64-tile IEEE-8500 feeder (~10.8 M local variables, the
  HBM-streaming path) to its stop -- identical iterations and status, bitwise
  x / z / lambda, bitwise max_local_infeasibility, trace within 1e-9;
- configs[4]: all 4096 IEEE-123 load scenarios -- every scenario's iteration
  count, status, objective (1e-12), infeasibility and x / z / lambda
  bitwise; the residual trace on a 64-scenario sample.

Both take minutes of oracle time (all host cores).
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest

from oracle import oracle_py as O
from paper_2501_08293_b200 import dopf
from test_gpu_parity import assert_same, assert_same_maxinf

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CORES = os.cpu_count() or 1


@pytest.mark.timeout(1800)
def test_tiled64_full_solve_parity():
    f = dopf.tiled_feeder("ieee8500", 64, 850064)   # bench.py --config tiled
    _, _, model = dopf.load_model(f, workers=CORES)
    model.precompute(CORES)
    s = dopf.CudaSolver(0)
    s.upload(model)
    assert s.info()["sync"] == "stream-graph"
    settings = dopf.Settings()
    gpu = s.solve(settings)
    assert gpu.status == dopf.CONVERGED
    ref = O.solve(model, dopf.Settings(workers=CORES))
    assert_same(gpu, ref, bitwise=True)


@pytest.mark.timeout(2400)
def test_batch4096_parity():
    from paper_2501_08293_b200 import scenarios
    from paper_2501_08293_b200.batch import BatchSolver
    models = scenarios.build_scenarios("ieee123", 123, range(4096))   # bench.py --config batch123
    settings = dopf.Settings()
    bs = BatchSolver(0)
    bs.upload(models)
    gpu = bs.solve(settings, trace=False)

    def oracle(m):
        return O.solve(m, dopf.Settings(workers=1))

    with cf.ThreadPoolExecutor(max_workers=CORES) as ex:  # ctypes releases the GIL
        refs = list(ex.map(oracle, models))
    its = set()
    for k, (g, r) in enumerate(zip(gpu, refs)):
        assert (g.status, g.iterations) == (r.status, r.iterations), k
        assert abs(g.objective - r.objective) <= 1e-12 * max(1.0, abs(r.objective)), k
        assert_same_maxinf(g, r)
        for a, b in ((g.x, r.x), (g.z, r.z), (g.lam, r.lam)):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), k
        assert (g.near_ties, g.first_near_tie) == (r.near_ties, r.first_near_tie), k
        its.add(g.iterations)
    assert len(its) > 100  # independent per-scenario stops
    # residual traces of a sample (a second, traced batch of 64 scenarios)
    sample = list(range(0, 4096, 64))
    bs64 = BatchSolver(0)
    bs64.upload([models[k] for k in sample])
    for k, g in zip(sample, bs64.solve(settings, trace=True)):
        assert_same(g, refs[k], bitwise=True)
