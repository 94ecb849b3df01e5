"""GPU parity: the sm_100a path through the C ABI (include/dopf_cuda.h) vs the
CPU oracle restating reference proj/src/admm.cpp:172-244.

Bar (BASELINE.json north_star): identical iteration count and status;
per-iterate x, z, lambda within 1e-9 relative (by construction the iterates
are bitwise identical -- asserted separately on the fixtures); final objective
within 1e-6 relative.
"""
import numpy as np
import pytest

from conftest import FIXTURES, fixture_path
from oracle import oracle_py as O
from paper_2501_08293_b200 import dopf

pytestmark = pytest.mark.gpu

REL = 1e-9
OBJ_REL = 1e-6


def rel_err(a, b):
    scale = max(1.0, float(np.max(np.abs(b)))) if b.size else 1.0
    return float(np.max(np.abs(a - b))) / scale if b.size else 0.0


def assert_same(gpu, ref, bitwise=False):
    assert gpu.status == ref.status
    assert gpu.iterations == ref.iterations
    for name, a, b in (("x", gpu.x, ref.x), ("z", gpu.z, ref.z), ("lambda", gpu.lam, ref.lam)):
        if bitwise:
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (name, rel_err(a, b))
        assert rel_err(a, b) <= REL, name
    assert abs(gpu.objective - ref.objective) <= OBJ_REL * max(1.0, abs(ref.objective))
    # residual trace: tree vs sequential summation, ulp-level only
    np.testing.assert_allclose(gpu.trace[:, 1:], ref.trace[:, 1:], rtol=1e-9, atol=1e-13)
    # max over iterations of ||A_s z_s - b_s||_inf (admm.cpp:203-205, 219-220):
    # the same sequential-j row sums on bitwise-equal z, and a max is
    # order-free -- so the value is bitwise equal, not just small
    assert_same_maxinf(gpu, ref)
    # stop tests within 1e-12 of flipping: none on these inputs, on either side
    assert (gpu.near_ties, gpu.first_near_tie) == (ref.near_ties, ref.first_near_tie)


def assert_same_maxinf(gpu, ref):
    a, b = np.float64(gpu.max_local_infeasibility), np.float64(ref.max_local_infeasibility)
    assert a.view(np.uint64) == b.view(np.uint64), (float(a), float(b))


def model_of_fixture(name):
    _, ls, model = dopf.load_model(fixture_path(name))
    model.precompute()
    return ls, model


@pytest.fixture(scope="module")
def solver():
    return dopf.CudaSolver(0)


@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("eps", [1e-3, 1e-4])
def test_fixture_solve_matches_oracle_bitwise(solver, name, eps):
    _, model = model_of_fixture(name)
    settings = dopf.Settings(rho=100.0, eps_rel=eps)
    solver.upload(model)
    gpu = solver.solve(settings)
    ref = O.solve(model, settings)
    assert gpu.status == dopf.CONVERGED
    assert_same(gpu, ref, bitwise=True)


def assert_snapshots_bitwise(gpu, ref, ts):
    for t in ts:
        g, r = gpu.snapshots[t], ref.snapshots[t]
        for k in ("x", "z", "z_prev", "lambda"):
            assert np.array_equal(g[k].view(np.uint64), r[k].view(np.uint64)), (t, k)


@pytest.mark.parametrize("name", FIXTURES)
def test_per_iterate_parity(name):
    """Every iterate t of the solve (parity mode: the device loop records the
    state after each iteration itself, reference record_iterates,
    admm.cpp:228-229): x, z, z_prev, lambda bitwise equal to the oracle's."""
    _, model = model_of_fixture(name)
    st = dopf.Settings(eps_rel=1e-12, max_iter=300)
    s = dopf.CudaSolver(0)
    s.set_path("resident")
    s.upload(model)
    gpu = s.solve(st, snapshots=st.max_iter)
    ts = list(range(1, gpu.iterations + 1))
    ref = O.solve(model, st, snap_iters=ts)
    assert (gpu.iterations, gpu.status) == (ref.iterations, ref.status)
    assert sorted(gpu.snapshots) == ts
    assert_snapshots_bitwise(gpu, ref, ts)


@pytest.mark.parametrize("shape,seed,T,every", [("ieee123", 123, 1000, 1), ("ieee8500", 8500, 200, 7)])
def test_per_iterate_parity_synthetic(shape, seed, T, every):
    f = dopf.synthetic_feeder(shape, seed)
    _, _, model = dopf.load_model(f, workers=4)
    model.precompute(4)
    st = dopf.Settings(max_iter=T)
    s = dopf.CudaSolver(0)
    s.upload(model)
    gpu = s.solve(st, snapshots=T)
    ts = sorted(set(range(1, gpu.iterations + 1, every)) | {gpu.iterations})
    ref = O.solve(model, dopf.Settings(max_iter=T, workers=4), snap_iters=ts)
    assert (gpu.iterations, gpu.status) == (ref.iterations, ref.status)
    assert_snapshots_bitwise(gpu, ref, ts)


@pytest.mark.parametrize("src", ["two_bus_delta", "four_bus_delta", "ieee123"])
def test_per_iterate_parity_streaming_path(src):
    """Parity mode on the HBM-streaming path (stream-ordered iterations with
    a snapshot copy after each): every iterate bitwise equal to the oracle."""
    if src == "ieee123":
        _, _, model = dopf.load_model(dopf.synthetic_feeder("ieee123", 123), workers=4)
        model.precompute(4)
        st = dopf.Settings(max_iter=300)
    else:
        _, model = model_of_fixture(src)
        st = dopf.Settings(eps_rel=1e-12, max_iter=300)
    s = dopf.CudaSolver(0)
    s.set_path("stream")
    s.upload(model)
    gpu = s.solve(st, snapshots=st.max_iter)
    ts = list(range(1, gpu.iterations + 1))
    ref = O.solve(model, st, snap_iters=ts)
    assert (gpu.iterations, gpu.status) == (ref.iterations, ref.status)
    assert sorted(gpu.snapshots) == ts
    assert_snapshots_bitwise(gpu, ref, ts)


def test_iteration_limit_is_a_status(solver):
    _, model = model_of_fixture("two_bus")
    solver.upload(model)
    res = solver.solve(dopf.Settings(eps_rel=1e-12, max_iter=10))
    assert res.status == dopf.ITERATION_LIMIT
    assert res.iterations == 10 and res.trace.shape == (10, 6)
    lo, hi = model.arr("x_lo"), model.arr("x_hi")
    assert np.all(res.x >= lo) and np.all(res.x <= hi)


def test_invalid_settings_raise(solver):
    _, model = model_of_fixture("single_bus")
    solver.upload(model)
    for bad in (dopf.Settings(rho=0.0), dopf.Settings(eps_rel=0.0), dopf.Settings(max_iter=0)):
        with pytest.raises(ValueError):
            solver.solve(bad)


@pytest.mark.parametrize("shape,seed", [("ieee13", 13), ("ieee123", 123)])
def test_synthetic_feeder_parity(solver, shape, seed):
    f = dopf.synthetic_feeder(shape, seed)
    _, _, model = dopf.load_model(f, workers=4)
    model.precompute(4)
    settings = dopf.Settings()
    solver.upload(model)
    gpu = solver.solve(settings)
    ref = O.solve(model, settings)
    assert_same(gpu, ref, bitwise=True)


def test_ieee8500_first_iterations_bitwise(solver):
    f = dopf.synthetic_feeder("ieee8500", 8500)
    _, _, model = dopf.load_model(f, workers=8)
    model.precompute(8)
    settings = dopf.Settings(eps_rel=1e-12, max_iter=60)
    solver.upload(model)
    info = solver.info()
    assert info["resident"]
    gpu = solver.solve(settings)
    ref = O.solve(model, settings)
    assert_same(gpu, ref, bitwise=True)


def test_batch_of_scenarios(solver):
    base = dopf.synthetic_feeder("ieee13", 13)
    models = []
    for k in range(6):
        f = dopf.scale_loads(base, 4096 + k)
        _, _, m = dopf.load_model(f)
        m.precompute()
        models.append(m)
    settings = dopf.Settings(eps_rel=1e-3)
    results = solver_batch(models, settings)
    for m, gpu in zip(models, results):
        ref = O.solve(m, settings)
        assert_same(gpu, ref, bitwise=True)


def solver_batch(models, settings):
    from paper_2501_08293_b200.batch import BatchSolver
    bs = BatchSolver(0)
    bs.upload(models)
    return bs.solve(settings)


@pytest.mark.timeout(600)
def test_tuned_partition_keeps_iterates_bitwise():
    """The slack-tuned resident split (dopf_cuda_tune_partition) changes only
    which CTA holds which subsystems: IEEE-8500 to convergence stays bitwise
    equal to the oracle, and the tuned split is not slower than the default."""
    f = dopf.synthetic_feeder("ieee8500", 8500)
    _, _, model = dopf.load_model(f, workers=8)
    model.precompute(8)
    s = dopf.CudaSolver(0)
    s.upload(model)
    base = min(s.solve(dopf.Settings(), outputs=False).timings["solve"] for _ in range(3))
    per = s.tune_partition(model, dopf.Settings(), rounds=6)
    gpu = s.solve(dopf.Settings())
    ref = O.solve(model, dopf.Settings(workers=8))
    assert_same(gpu, ref, bitwise=True)
    assert per * gpu.iterations <= base * 1.02
    s.upload(model)  # a same-structure re-upload keeps the tuned split
    assert_same(s.solve(dopf.Settings()), ref, bitwise=True)
    import ctypes as C
    w = (C.c_double * 256)()
    assert s._lib.dopf_cuda_block_weights(s._h, w, 256) == s.info()["blocks"]
    # another structure on the same context: the shares tuned for IEEE-8500 are dropped
    _, _, other = dopf.load_model(dopf.synthetic_feeder("ieee8500", 8501), workers=8)
    other.precompute(8)
    s.upload(other)
    assert s._lib.dopf_cuda_block_weights(s._h, w, 256) == 0
    assert_same(s.solve(dopf.Settings(max_iter=200)), O.solve(other, dopf.Settings(max_iter=200, workers=8)),
                bitwise=True)


@pytest.mark.timeout(600)
def test_ieee8500_full_solve_bitwise(solver):
    """The paper's largest case to convergence: identical iteration count and
    bitwise-identical x, z, lambda (the multi-block exchange protocol at scale)."""
    f = dopf.synthetic_feeder("ieee8500", 8500)
    _, _, model = dopf.load_model(f, workers=8)
    model.precompute(8)
    settings = dopf.Settings()
    solver.upload(model)
    gpu = solver.solve(settings)
    ref = O.solve(model, dopf.Settings(workers=8))
    assert gpu.status == dopf.CONVERGED
    assert_same(gpu, ref, bitwise=True)
    again = solver.solve(settings)  # run-to-run determinism of the device loop
    assert again.iterations == gpu.iterations
    assert np.array_equal(again.trace, gpu.trace)


@pytest.mark.parametrize("tune", ["0", "1"])
def test_cpp_dropin_program(tune):
    """Reference-style C++ caller of dopf::solve linked against libdopf_cuda.so
    (DOPF_TUNE=1: the drop-in also tunes the split on its first call per
    structure; the program's bitwise checks must hold either way)."""
    import os
    import subprocess

    from conftest import ROOT
    from paper_2501_08293_b200 import build
    proc = subprocess.run([build.DROPIN_TEST, os.path.join(ROOT, "tests", "golden", "fixtures")],
                          capture_output=True, text=True, timeout=600, env={**os.environ, "DOPF_TUNE": tune})
    assert proc.returncode == 0, proc.stdout + proc.stderr
    assert "PASS" in proc.stdout


@pytest.mark.timeout(900)
def test_batch_ieee123_scenarios_bitwise():
    """Config 5 shape: independent IEEE-123 load scenarios, each a multi-CTA
    cluster instance with its own iteration count, bitwise equal to the oracle."""
    from paper_2501_08293_b200 import scenarios
    models = scenarios.build_scenarios("ieee123", 123, range(6))
    settings = dopf.Settings()
    results = solver_batch(models, settings)
    its = set()
    for m, gpu in zip(models, results):
        ref = O.solve(m, dopf.Settings(workers=8))
        assert_same(gpu, ref, bitwise=True)
        its.add(gpu.iterations)
    assert len(its) > 1  # scenarios really converge independently


@pytest.mark.timeout(600)
def test_batch_persistent_groups_several_instances_per_group_bitwise():
    """Batches run as persistent CTA groups (admm_groups): with 100 IEEE-123
    scenarios over 37 groups of 4 CTAs every group solves 2-3 instances one
    after another in the same CTAs -- each still bitwise equal to the oracle
    (iterations, status, x / z / lambda, max_local_infeasibility, trace)."""
    import concurrent.futures as cf
    import os
    from paper_2501_08293_b200 import scenarios
    models = scenarios.build_scenarios("ieee123", 123, range(100))
    settings = dopf.Settings()
    results = solver_batch(models, settings)
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        refs = list(ex.map(lambda m: O.solve(m, dopf.Settings(workers=1)), models))
    for gpu, ref in zip(results, refs):
        assert_same(gpu, ref, bitwise=True)


@pytest.mark.timeout(600)
def test_tuned_batch_split_keeps_iterates_bitwise():
    """A batch split tuned on a scenario sample (dopf_cuda_tune_partition_batch)
    and a tuned 4-CTA single IEEE-123 instance: every scenario still bitwise
    equal to the oracle."""
    import concurrent.futures as cf
    import os
    from paper_2501_08293_b200 import scenarios
    from paper_2501_08293_b200.batch import BatchSolver
    models = scenarios.build_scenarios("ieee123", 123, range(60))
    bs = BatchSolver(0)
    bs.tune_partition(models[:20], dopf.Settings(), rounds=4)
    bs.upload(models)
    results = bs.solve(dopf.Settings())
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        refs = list(ex.map(lambda m: O.solve(m, dopf.Settings(workers=1)), models))
    for gpu, ref in zip(results, refs):
        assert_same(gpu, ref, bitwise=True)
    s = dopf.CudaSolver(0)
    s.tune_partition(models[0], dopf.Settings(), rounds=4)
    assert s.info()["sync"] == "cluster"
    assert_same(s.solve(dopf.Settings()), refs[0], bitwise=True)


# ------------------------------------------------------------ HBM-streaming path


@pytest.fixture(scope="module")
def stream_solver():
    s = dopf.CudaSolver(0)
    s.set_path("stream")
    return s


@pytest.mark.parametrize("name", FIXTURES)
def test_stream_path_fixtures_bitwise(stream_solver, name):
    _, model = model_of_fixture(name)
    settings = dopf.Settings(rho=100.0, eps_rel=1e-4)
    stream_solver.upload(model)
    assert stream_solver.info()["sync"] == "stream-graph"
    gpu = stream_solver.solve(settings)
    ref = O.solve(model, settings)
    assert gpu.status == dopf.CONVERGED
    assert_same(gpu, ref, bitwise=True)


@pytest.mark.parametrize("shape,seed,max_iter", [("ieee123", 123, 50000), ("ieee8500", 8500, 200)])
def test_stream_path_synthetic_bitwise(stream_solver, shape, seed, max_iter):
    f = dopf.synthetic_feeder(shape, seed)
    _, _, model = dopf.load_model(f, workers=8)
    model.precompute(8)
    settings = dopf.Settings(max_iter=max_iter)
    stream_solver.upload(model)
    gpu = stream_solver.solve(settings)
    ref = O.solve(model, dopf.Settings(max_iter=max_iter, workers=8))
    assert_same(gpu, ref, bitwise=True)


@pytest.mark.timeout(900)
def test_tiled_feeder_auto_streams_bitwise():
    """Tiled IEEE-8500 copies under one root (config 4 shape): too large for
    shared-memory residency, so the auto path streams from HBM."""
    f = dopf.tiled_feeder("ieee8500", 4, 850064)
    _, _, model = dopf.load_model(f, workers=8)
    model.precompute(8)
    s = dopf.CudaSolver(0)
    s.upload(model)
    assert s.info()["sync"] == "stream-graph"
    settings = dopf.Settings(max_iter=300)
    gpu = s.solve(settings)
    ref = O.solve(model, dopf.Settings(max_iter=300, workers=8))
    assert_same(gpu, ref, bitwise=True)


# ------------------------------------------------------------ GPU precompute (row f2)


@pytest.mark.parametrize("source", FIXTURES + ["ieee123", "ieee8500"])
def test_gpu_precompute_bitwise_equals_host(solver, source):
    if source in FIXTURES:
        _, _, host = dopf.load_model(fixture_path(source))
        _, _, gpu = dopf.load_model(fixture_path(source))
    else:
        f = dopf.synthetic_feeder(source, 123 if source == "ieee123" else 8500)
        _, _, host = dopf.load_model(f, workers=4)
        _, _, gpu = dopf.load_model(f, workers=4)
    host.precompute(4)
    gpu.precompute_gpu(solver)
    for name in ("P", "v", "inv_copy", "csr_ptr", "csr_copy"):
        assert np.array_equal(host.arr(name), gpu.arr(name)), name


def test_gpu_precompute_flags_singular_subsystem(solver):
    m = dopf.single_sub_model([[1.0, 0, 0], [1.0, 0, 0]], [1.0, 1.0], np.zeros(3), [-np.inf] * 3,
                              [np.inf] * 3)
    with pytest.raises(dopf.SingularSubsystemError):
        m.precompute_gpu(solver)


def test_reupload_same_structure_fast_path_bitwise(solver):
    """Scenarios share the structure: the second and later uploads copy raw
    values and scatter them on the GPU (cached plan) -- still bitwise."""
    from paper_2501_08293_b200 import scenarios
    models = scenarios.build_scenarios("ieee123", 123, range(3))
    settings = dopf.Settings()
    for m in models + models[:1]:
        solver.upload(m)
        gpu = solver.solve(settings)
        ref = O.solve(m, dopf.Settings(workers=8))
        assert_same(gpu, ref, bitwise=True)


def test_stream_reupload_same_structure_fast_path_bitwise():
    """Streaming path: a same-structure re-upload skips the host layout build
    (raw values + device gather over the cached maps) -- still bitwise."""
    from paper_2501_08293_b200 import scenarios
    models = scenarios.build_scenarios("ieee123", 123, range(3))
    s = dopf.CudaSolver(0)
    s.set_path("stream")
    settings = dopf.Settings()
    for m in models + models[:1]:
        s.upload(m)
        gpu = s.solve(settings)
        ref = O.solve(m, dopf.Settings(workers=8))
        assert_same(gpu, ref, bitwise=True)


# ------------------------------------------------------------ certification (row f4)


@pytest.mark.parametrize("source", ["two_bus", "four_bus_delta", "ieee8500"])
def test_gpu_certify_and_reconstruct_match_host_checks(solver, source):
    if source.startswith("ieee"):
        f = dopf.synthetic_feeder(source, 8500)
        _, ls, model = dopf.load_model(f, workers=8)
        model.precompute(8)
    else:
        _, ls, model = dopf.load_model(fixture_path(source))
        model.precompute()
    solver.upload(model)
    res = solver.solve(dopf.Settings(eps_rel=1e-4))
    rebuilt = dopf.reconstruct_centralized(model, res.x, res.z, solver)
    assert np.array_equal(rebuilt, O.reconstruct_centralized(model, res.x, res.z))
    for x in (rebuilt, res.x, np.zeros(ls.cols)):
        gpu, host = dopf.check_feasibility(ls, x, solver), O.check_feasibility(ls, x)
        for k in ("max_equality_violation", "max_bound_violation", "worst_row", "worst_col", "objective"):
            assert gpu[k] == host[k], (k, gpu[k], host[k])


# ------------------------------------------------------------ exact division by rho


@pytest.mark.parametrize("rho", [100.0, 1.0, 3.0, 0.7, 1e-3, 12345.678, 2.0 ** -400, 2.0 ** 600])
def test_div_rho_is_the_ieee_quotient(solver, rho):
    """The kernels divide by rho through RN(1/rho) plus two exact-residual
    corrections (div_rho.cuh); the result must be the IEEE quotient bit for
    bit, over random magnitudes, both signs, zeros, subnormals, huge values
    and non-finite inputs."""
    import ctypes as C
    from paper_2501_08293_b200 import _native as N
    rng = np.random.default_rng(20251017)
    n = 1 << 21
    mant = rng.uniform(1.0, 2.0, n)
    expo = rng.integers(-1074, 1023, n)
    a = np.ldexp(mant, expo) * rng.choice([-1.0, 1.0], n)
    a[: n // 2] = rng.standard_normal(n // 2) * 10.0 ** rng.uniform(-8, 8, n // 2)  # the ADMM range
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                        1.7976931348623157e308, -1.7976931348623157e308, 1.0, -1.0, rho, -rho])
    a[: special.size] = special
    out = np.empty_like(a)
    lib = N.cuda()
    rc = lib.dopf_cuda_div_rho_check(solver._h, a.ctypes.data_as(C.POINTER(C.c_double)), n, rho,
                                     out.ctypes.data_as(C.POINTER(C.c_double)))
    assert rc == 0
    with np.errstate(all="ignore"):
        ref = a / rho
    same = (out.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(out) & np.isnan(ref))
    assert same.all(), (a[~same][:5], out[~same][:5], ref[~same][:5])


@pytest.mark.parametrize("stage_kb,ctas,direct", [(1, "2", True), (8, "2", True), (16, "3", True),
                                                  (32, "3", False)])
def test_stream_direct_and_staged_chunk_mix_bitwise(monkeypatch, stage_kb, ctas, direct):
    """Small pipeline stages push many chunks onto the direct-load kernel
    (image read from HBM) beside the staged kernel; 3 staged CTAs per SM
    exercises the other residency. Both chunk kernels share one iteration
    routine and must stay bitwise equal to the oracle."""
    monkeypatch.setenv("DOPF_STAGE_KB", str(stage_kb))
    monkeypatch.setenv("DOPF_STAGED_CTAS", ctas)
    f = dopf.synthetic_feeder("ieee8500", 8500)
    _, _, model = dopf.load_model(f, workers=8)
    model.precompute(8)
    s = dopf.CudaSolver(0)
    s.set_path("stream")
    s.upload(model)
    info = s.stream_info()
    assert (info["direct_chunks"] > 0) == direct, info
    if stage_kb > 1:
        assert info["staged_chunks"] > 0, info
    else:  # every chunk direct: no staged CTAs, partial slots / fold count of the direct kernel only
        assert info["staged_chunks"] == 0 and info["staged_ctas"] == 0, info
    assert info["stage_bytes"] == stage_kb * 1024
    settings = dopf.Settings(max_iter=150)
    gpu = s.solve(settings)
    ref = O.solve(model, dopf.Settings(max_iter=150, workers=8))
    assert_same(gpu, ref, bitwise=True)


@pytest.mark.parametrize("path", ["resident", "stream"])
def test_pinned_inputs_and_results_bitwise(path):
    """Page-locked model arrays (dopf_cuda_pin_model) and result buffers: the
    uploads take the DMA path and results are copied straight into the
    caller's arrays -- same bits as the oracle."""
    import ctypes as C
    from paper_2501_08293_b200 import _native as N
    f = dopf.synthetic_feeder("ieee123", 123)
    _, _, model = dopf.load_model(f, workers=4)
    model.precompute(4)
    s = dopf.CudaSolver(0)
    s.set_path(path)
    s.pin(model)
    s.pin(model)  # pinning twice is a no-op
    settings = dopf.Settings()
    ref = O.solve(model, dopf.Settings(workers=8))
    v = model.view()
    x, z, lam = np.zeros(v.n), np.zeros(v.N_z), np.zeros(v.N_z)
    tr = np.zeros((settings.max_iter, 6))
    for a in (x, z, lam, tr):
        s.pin_array(a)
    lib = N.cuda()
    for _ in range(2):  # second upload: same structure, values-only path
        assert lib.dopf_cuda_upload(s._h, C.byref(v)) == 0
        r = N.ResultView_t()
        r.x = x.ctypes.data_as(C.POINTER(C.c_double))
        r.z = z.ctypes.data_as(C.POINTER(C.c_double))
        r.lambda_ = lam.ctypes.data_as(C.POINTER(C.c_double))
        r.trace = tr.ctypes.data_as(C.POINTER(C.c_double))
        assert lib.dopf_cuda_solve(s._h, C.byref(settings.to_c()), C.byref(r)) == 0
        assert r.iterations == ref.iterations and r.status == ref.status
        for a, b in ((x, ref.x), (z, ref.z), (lam, ref.lam)):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
        np.testing.assert_allclose(tr[:r.iterations, 1:], ref.trace[:, 1:], rtol=1e-9, atol=1e-13)
    s.unpin(model)


def test_stream_path_run_to_run_deterministic(stream_solver):
    """The streaming path's residual partials are folded in a fixed order
    (whichever chunk CTA finishes last): two solves give the same trace bits."""
    f = dopf.synthetic_feeder("ieee8500", 8500)
    _, _, model = dopf.load_model(f, workers=8)
    model.precompute(8)
    stream_solver.upload(model)
    settings = dopf.Settings(max_iter=300)
    a = stream_solver.solve(settings)
    b = stream_solver.solve(settings)
    assert a.iterations == b.iterations
    assert np.array_equal(a.trace.view(np.uint64), b.trace.view(np.uint64))
    assert a.objective == b.objective and a.max_local_infeasibility == b.max_local_infeasibility
