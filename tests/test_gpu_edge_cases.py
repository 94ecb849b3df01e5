"""GPU parity on the reference's edge cases and settings range.

- rho sweep: every other GPU test runs at the paper's rho = 100; the kernels
  divide by rho through div_rho (div_rho.cuh) and precompute c / rho, so other
  penalties must be bitwise too (both device paths).
- the square, fully determined model of proj/tests/test_admm.cpp:328-344;
- subsystems without rows (m_s = 0, P = I: proj/src/admm.cpp:41-46), alone
  and mixed with constrained ones;
- settings rejected at the C ABI itself (code 1 = std::invalid_argument,
  admm.cpp:173-175), not only by the Python mirror;
- the stop-test near-tie guard (stop_test.cuh) on a constructed tie.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import FIXTURES, fixture_path
from oracle import oracle_py as O
from paper_2501_08293_b200 import _native as N
from paper_2501_08293_b200 import dopf
from test_gpu_parity import assert_same

pytestmark = pytest.mark.gpu

INF = np.inf
RHOS = [1.0, 0.7, 1e3]


@pytest.fixture(scope="module", params=["resident", "stream"])
def solver(request):
    s = dopf.CudaSolver(0)
    s.set_path(request.param)
    return s


def fixture_model(name):
    _, _, m = dopf.load_model(fixture_path(name))
    m.precompute()
    return m


@pytest.mark.parametrize("rho", RHOS)
@pytest.mark.parametrize("name", FIXTURES)
def test_rho_sweep_fixtures_bitwise(solver, name, rho):
    m = fixture_model(name)
    settings = dopf.Settings(rho=rho, eps_rel=1e-4, max_iter=20000)
    solver.upload(m)
    gpu = solver.solve(settings)
    ref = O.solve(m, settings)
    assert_same(gpu, ref, bitwise=True)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("rho", RHOS)
def test_rho_sweep_ieee123_bitwise(solver, rho):
    f = dopf.synthetic_feeder("ieee123", 123)
    _, _, m = dopf.load_model(f, workers=4)
    m.precompute(4)
    settings = dopf.Settings(rho=rho, max_iter=6000)
    solver.upload(m)
    gpu = solver.solve(settings)
    ref = O.solve(m, dopf.Settings(rho=rho, max_iter=6000, workers=8))
    assert_same(gpu, ref, bitwise=True)


@pytest.mark.parametrize("rho", [0.7, 1e3])
def test_rho_sweep_ieee8500_bitwise(solver, rho):
    f = dopf.synthetic_feeder("ieee8500", 8500)
    _, _, m = dopf.load_model(f, workers=8)
    m.precompute(8)
    settings = dopf.Settings(rho=rho, max_iter=200)
    solver.upload(m)
    gpu = solver.solve(settings)
    ref = O.solve(m, dopf.Settings(rho=rho, max_iter=200, workers=8))
    assert_same(gpu, ref, bitwise=True)


def test_square_model_converges_to_unique_point(solver):
    """test_admm.cpp:328-344: A square and invertible -> P = 0, z = v = A^-1 b;
    x is pinned to the unique solution within 1e-10."""
    a = np.array([[2.0, 1.0], [1.0, 3.0]])
    sol = np.array([0.4, 0.7])
    m = dopf.single_sub_model(a, a @ sol, [1.0, 0.0], [-10, -10], [10, 10])
    m.precompute()
    settings = dopf.Settings(eps_rel=1e-8, max_iter=100)
    solver.upload(m)
    gpu = solver.solve(settings)
    ref = O.solve(m, settings)
    assert gpu.status == dopf.CONVERGED
    assert np.abs(gpu.x - sol).max() <= 1e-10
    assert_same(gpu, ref, bitwise=True)


def no_row_models():
    # one subsystem without rows: P = I, v = 0 (admm.cpp:41-46)
    alone = dopf.single_sub_model(np.zeros((0, 3)), [], [1.0, -2.0, 0.5], [-1, -1, 0], [1, 1, 2])
    # m_s = 0 subsystems sharing columns with constrained ones
    mixed = dopf.model_from_arrays(
        [(np.array([[1.0, 1.0]]), [1.0], [0, 1]),
         (np.zeros((0, 2)), [], [1, 2]),
         (np.array([[1.0, -1.0], [0.5, 2.0]]), [0.2, 1.0], [2, 3]),
         (np.zeros((0, 3)), [], [0, 3, 4])],
        [0.3, -0.1, 0.2, 0.4, -0.5], [-2] * 5, [2] * 5)
    return {"alone": alone, "mixed": mixed}


@pytest.mark.parametrize("kind", ["alone", "mixed"])
@pytest.mark.parametrize("rho", [100.0, 0.7])
def test_subsystems_without_rows_bitwise(solver, kind, rho):
    m = no_row_models()[kind]
    m.precompute()
    for eps, max_iter in ((1e-6, 5000), (1e-12, 37)):
        settings = dopf.Settings(rho=rho, eps_rel=eps, max_iter=max_iter)
        solver.upload(m)
        gpu = solver.solve(settings)
        ref = O.solve(m, settings)
        assert_same(gpu, ref, bitwise=True)
        assert gpu.max_local_infeasibility == ref.max_local_infeasibility


@pytest.mark.parametrize("bad", [dict(rho=0.0), dict(rho=-1.0), dict(rho=float("nan")), dict(eps_rel=0.0),
                                 dict(eps_rel=float("nan")), dict(max_iter=0)])
def test_invalid_settings_rejected_by_the_c_abi(solver, bad):
    """The C ABI validates settings itself (admm.cpp:173-175): code 1, the
    std::invalid_argument of dopf::solve, and a message naming the setting."""
    m = fixture_model("single_bus")
    solver.upload(m)
    s = dopf.Settings(**bad).to_c()
    r = N.ResultView_t()
    lib = N.cuda()
    for fn in (lib.dopf_cuda_solve, lib.dopf_cuda_solve_device):
        assert fn(solver._h, C.byref(s), C.byref(r)) == N_INVALID
        msg = lib.dopf_cuda_last_error(solver._h).decode()
        assert list(bad)[0] in msg, msg
    assert lib.dopf_cuda_solve(solver._h, None, C.byref(r)) == N_INVALID


N_INVALID = 1  # DOPF_ERR_INVALID_ARGUMENT


def constructed_tie(m, horizon=400):
    """eps_rel that puts the stop test of some iteration t0 exactly on its
    threshold, t0 being the first iteration the looser test would accept: the
    last record low of the required tolerance max(pres / max(||Bx||, ||z||),
    dres / ||lambda||) over the first `horizon` iterations of an
    effectively-never-stopping run."""
    tiny = 1e-14
    probe = O.solve(m, dopf.Settings(eps_rel=tiny, max_iter=horizon))
    tr = probe.trace
    need = np.maximum(tr[:, 1] / (tr[:, 3] / tiny), tr[:, 2] / (tr[:, 4] / tiny))
    lows = [t for t in range(1, len(need) + 1) if need[t - 1] < need[: t - 1].min(initial=np.inf)]
    t0 = lows[-1]
    return float(need[t0 - 1]), t0


def test_near_tie_flag_on_a_constructed_tie(solver):
    """Both the oracle and the device flag the constructed tie at t0 (and no
    earlier iteration), whatever the ulp-level outcome of the comparison."""
    m = fixture_model("four_bus_delta")
    eps, t0 = constructed_tie(m)
    assert t0 > 20
    settings = dopf.Settings(eps_rel=eps, max_iter=t0 + 50)
    ref = O.solve(m, settings)
    solver.upload(m)
    gpu = solver.solve(settings)
    assert ref.first_near_tie == t0 and ref.near_ties >= 1, (t0, ref.first_near_tie, ref.iterations)
    assert gpu.first_near_tie == t0 and gpu.near_ties >= 1, (t0, gpu.first_near_tie, gpu.iterations)
    assert min(gpu.iterations, ref.iterations) >= t0


def wide_subsystem_model(n=150, m=100, seed=5):
    """One subsystem with n_s = 150 >= 128 columns: beyond the resident
    kernel's packed row metadata, within a streaming chunk."""
    rng = np.random.default_rng(seed)
    a = rng.normal(size=(m, n))
    b = a @ rng.normal(size=n)
    lo = np.where(rng.random(n) < 0.5, -1.0, -INF)
    hi = np.where(rng.random(n) < 0.5, 1.0, INF)
    mdl = dopf.single_sub_model(a, b, rng.normal(size=n), lo, hi)
    mdl.precompute()
    return mdl


def test_auto_path_falls_back_to_streaming_beyond_resident_limits():
    m = wide_subsystem_model()
    s = dopf.CudaSolver(0)
    s.upload(m)  # auto: the resident plan is rejected, the streaming path takes it
    assert s.info()["sync"] == "stream-graph"
    st = dopf.Settings(max_iter=400)
    assert_same(s.solve(st), O.solve(m, st), bitwise=True)
    forced = dopf.CudaSolver(0)
    forced.set_path("resident")
    with pytest.raises(ValueError):
        forced.upload(m)


@pytest.mark.parametrize("n,m", [(700, 300), (1024, 1000)])
def test_hub_subsystem_wider_than_a_chunk_streams_bitwise(n, m):
    """A subsystem wider than 512 columns (a hub bus: the root of a feeder
    tiled > 85 times) runs on a 1024-thread direct-load CTA."""
    mdl = wide_subsystem_model(n, m, seed=n)
    s = dopf.CudaSolver(0)
    s.upload(mdl)
    assert s.info()["sync"] == "stream-graph"
    st = dopf.Settings(max_iter=200)
    assert_same(s.solve(st), O.solve(mdl, st), bitwise=True)


@pytest.mark.slow
@pytest.mark.timeout(1200)
def test_tiled_feeder_beyond_85_tiles_bitwise():
    """96 IEEE-8500 tiles on one root bus: the root subsystem is ~580 columns
    wide (rejected by both paths before); first iterations bitwise."""
    import os
    f = dopf.tiled_feeder("ieee8500", 96, 850096)
    _, _, model = dopf.load_model(f, workers=os.cpu_count() or 1)
    model.precompute(os.cpu_count() or 1)
    ns = np.diff(model.z_offsets)
    assert ns.max() > 512
    s = dopf.CudaSolver(0)
    s.upload(model)
    st = dopf.Settings(max_iter=12)
    ref = O.solve(model, dopf.Settings(max_iter=12, workers=os.cpu_count() or 1))
    assert_same(s.solve(st), ref, bitwise=True)


def test_block_stats_describe_the_resident_layout():
    """dopf_cuda_block_stats (load-balance diagnostics) agrees with the model:
    every row in exactly one block, sums of n_s over rows = sum n_s^2."""
    f = dopf.synthetic_feeder("ieee123", 123)
    _, _, m = dopf.load_model(f, workers=4)
    m.precompute(4)
    s = dopf.CudaSolver(0)
    s.upload(m)
    G = s.info()["blocks"]
    out = (N.i64 * (12 * G))()
    assert s._lib.dopf_cuda_block_stats(s._h, out, G) == 0
    st = np.array(out[:], dtype=np.int64).reshape(G, 12)
    ns = np.diff(m.z_offsets)
    assert st[:, 0].sum() == m.total_local_vars            # rows
    assert st[:, 11].sum() == int((ns.astype(np.int64) ** 2).sum())  # sum of n_s over rows
    assert (st[:, 10] >= 1).all()                             # longest per-thread chain


def test_tuning_is_a_noop_off_the_resident_path():
    """Split tuning on a streaming upload leaves the model untouched (0 returned)."""
    _, _, m = dopf.load_model(fixture_path("four_bus_delta"))
    m.precompute()
    s = dopf.CudaSolver(0)
    s.set_path("stream")
    assert s.tune_partition(m, dopf.Settings(), rounds=3) == 0.0
    assert s.info()["sync"] == "stream-graph"
    st = dopf.Settings(eps_rel=1e-4)
    assert_same(s.solve(st), O.solve(m, st), bitwise=True)


@pytest.mark.parametrize("seed", range(100, 112))
def test_random_radial_feeders_bitwise_both_paths(seed):
    """Random radial feeders (tests/feeder_gen.py, the ranges of the reference's
    test_util.hpp:77-172, 20-60 buses) through the whole pipeline and both
    device paths: iterations, status, x / z / lambda, infeasibility and near-tie
    counters identical to the oracle. Infeasible draws (a legitimate outcome,
    test_decompose.cpp:319-323) are skipped."""
    from feeder_gen import random_feeder
    f = dopf.parse_feeder(random_feeder(seed, n_buses=20 + (seed % 5) * 10))
    try:
        _, _, m = dopf.load_model(f)
        m.precompute()
    except (dopf.InfeasibleSubsystemError, dopf.SingularSubsystemError):
        pytest.skip("infeasible / singular draw")
    st = dopf.Settings(eps_rel=1e-4, max_iter=3000)
    ref = O.solve(m, st)
    for path in ("resident", "stream"):
        s = dopf.CudaSolver(0)
        s.set_path(path)
        s.upload(m)
        assert_same(s.solve(st), ref, bitwise=True)
