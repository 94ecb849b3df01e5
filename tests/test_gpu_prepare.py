"""Row f2 on the GPU: row_reduce (reference decompose.cpp:48-98,
reduce_subsystems :175-199) and the one-time operators (admm.cpp:31-88) of
many models in one batched call (dopf.prepare_gpu -> dopf_cuda_prepare),
bitwise against the host restatement that the CPU oracle iterates with --
including the reference's error behaviour (InfeasibleSubsystemError naming
the component, test_decompose.cpp:310-316)."""
import numpy as np
import pytest

from conftest import fixture_path
from paper_2501_08293_b200 import dopf, scenarios

pytestmark = pytest.mark.gpu

FIXTURES = ["single_bus", "two_bus", "two_bus_delta", "three_bus_transformer", "four_bus_delta"]


@pytest.fixture(scope="module")
def solver():
    return dopf.CudaSolver(0)


def partitioned(src):
    f = src if isinstance(src, dopf.Feeder) else dopf.parse_feeder_file(src)
    ls = dopf.assemble_centralized(f)
    return dopf.partition(ls, f)


def host_model(src, tol=1e-9):
    m = partitioned(src)
    m.reduce(tol, 4)
    m.precompute(4)
    return m


def assert_models_bitwise(g, h):
    assert g.S == h.S
    assert np.array_equal(g.arr("m_s"), h.arr("m_s"))
    assert np.array_equal(g.rows_before_reduction(), h.rows_before_reduction())
    for name in ("A", "b", "P", "v", "inv_copy", "csr_ptr", "csr_copy", "l2g", "z_offsets"):
        a, b = g.arr(name), h.arr(name)
        assert a.shape == b.shape, name
        assert np.array_equal(a.view(np.uint64) if a.dtype == np.float64 else a,
                              b.view(np.uint64) if b.dtype == np.float64 else b), name


@pytest.mark.parametrize("source", FIXTURES + ["ieee13", "ieee123", "ieee8500"])
def test_prepare_bitwise_equals_host(solver, source):
    src = fixture_path(source) if source in FIXTURES else \
        dopf.synthetic_feeder(source, {"ieee13": 13, "ieee123": 123, "ieee8500": 8500}[source])
    g = partitioned(src)
    secs = dopf.prepare_gpu([g], solver)
    assert secs["kernels_s"] > 0
    assert_models_bitwise(g, host_model(src))


def test_prepare_batch_of_scenarios_bitwise(solver):
    base = dopf.synthetic_feeder("ieee123", 123)
    fs = [dopf.scale_loads(base, scenarios.scenario_seed(123, k)) for k in range(40)]
    gs = [partitioned(f) for f in fs]
    dopf.prepare_gpu(gs, solver, chunk=16)  # three chunks, the last one partial
    for f, g in zip(fs, gs):
        assert_models_bitwise(g, host_model(f))


def test_build_scenarios_gpu_matches_host(solver):
    host = scenarios.build_scenarios("ieee123", 123, range(8))
    gpu = scenarios.build_scenarios("ieee123", 123, range(8), gpu=solver)
    for g, h in zip(gpu, host):
        assert_models_bitwise(g, h)


def random_rank_deficient(rng, m, n, r, ints):
    """m x n of rank <= r; integer entries (pivot ties everywhere) or reals."""
    if ints:
        base = rng.integers(-2, 3, size=(r, n)).astype(np.float64)
        mix = rng.integers(-1, 2, size=(m, r)).astype(np.float64)
    else:
        base = rng.normal(size=(r, n))
        mix = rng.normal(size=(m, r))
    a = mix @ base
    x0 = rng.normal(size=n)
    return a, a @ x0


@pytest.mark.parametrize("ints", [True, False])
def test_prepare_random_rank_deficient_bitwise(solver, ints):
    rng = np.random.default_rng(2501 + ints)
    gs, hs = [], []
    for _ in range(40):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(1, 30))
        r = int(rng.integers(1, min(m, n) + 1))
        a, b = random_rank_deficient(rng, m, n, r, ints)
        mk = lambda: dopf.single_sub_model(a, b, np.zeros(n), [-np.inf] * n, [np.inf] * n)
        gs.append(mk())
        h = mk()
        h.reduce()
        h.precompute()
        hs.append(h)
    dopf.prepare_gpu(gs, solver)
    for g, h in zip(gs, hs):
        assert_models_bitwise(g, h)


def test_prepare_subsystem_beyond_shared_memory(solver):
    """m x n = 120 x 200: the projector's work space (615 KB) exceeds shared
    memory, so every subsystem of the call runs on global scratch."""
    rng = np.random.default_rng(7)
    a, b = random_rank_deficient(rng, 150, 200, 120, False)
    mk = lambda: dopf.single_sub_model(a, b, np.zeros(200), [-np.inf] * 200, [np.inf] * 200)
    g, h = mk(), mk()
    h.reduce()
    h.precompute()
    dopf.prepare_gpu([g], solver)
    assert int(g.arr("m_s")[0]) == 120
    assert_models_bitwise(g, h)


def test_prepare_infeasible_names_the_component(solver):
    # contradictory rows (x1 = 1 and x1 = 2): the host raises
    # InfeasibleSubsystemError for the first failing subsystem in order
    ok = dopf.single_sub_model([[1.0, 1.0]], [1.0], np.zeros(2), [-np.inf] * 2, [np.inf] * 2)
    bad = dopf.single_sub_model([[1.0, 0.0], [2.0, 0.0]], [1.0, 4.0], np.zeros(2), [-np.inf] * 2,
                                [np.inf] * 2)
    with pytest.raises(dopf.InfeasibleSubsystemError) as host:
        bad.reduce()
    bad = dopf.single_sub_model([[1.0, 0.0], [2.0, 0.0]], [1.0, 4.0], np.zeros(2), [-np.inf] * 2,
                                [np.inf] * 2)
    with pytest.raises(dopf.InfeasibleSubsystemError) as gpu:
        dopf.prepare_gpu([ok, bad], solver)
    assert gpu.value.subsystem_id == host.value.subsystem_id == "s0"


def test_precompute_gpu_singular_names_the_component(solver):
    # unreduced duplicate rows: A A' is singular (the reference's guard)
    m = dopf.single_sub_model([[1.0, 0, 0], [1.0, 0, 0]], [1.0, 1.0], np.zeros(3), [-np.inf] * 3,
                              [np.inf] * 3)
    with pytest.raises(dopf.SingularSubsystemError) as e:
        m.precompute_gpu(solver)
    assert e.value.subsystem_id == "s0"


def test_prepared_model_solves_bitwise_like_host(solver):
    from oracle import oracle_py as O
    f = dopf.synthetic_feeder("ieee123", 123)
    g = partitioned(f)
    dopf.prepare_gpu([g], solver)
    s = dopf.CudaSolver(0)
    s.upload(g)
    st = dopf.Settings()
    gpu = s.solve(st)
    ref = O.solve(host_model(f), st)
    assert (gpu.status, gpu.iterations) == (ref.status, ref.iterations)
    assert np.array_equal(gpu.x.view(np.uint64), ref.x.view(np.uint64))
