"""Pins the CPU oracle (and the shared host precompute) to the reference's own
known answers. The C++ reference cannot be built here (Eigen3 and vendor/ are
absent), so these are the reference's tests restated:

  frozen LP objectives          proj/tests/test_oracle.cpp:23-29
  ADMM within 10 eps_rel        proj/tests/test_oracle.cpp:216-229
  precompute KATs               proj/tests/test_admm.cpp:53-111
  global / local / dual KATs    proj/tests/test_admm.cpp:113-270
  residual KATs                 proj/tests/test_admm.cpp:272-303
  init rule                     proj/tests/test_admm.cpp:305-326
  solve KATs                    proj/tests/test_admm.cpp:328-418
  acceptance criteria 1-7, 9    proj/tests/acceptance.cpp:89-393

Random trials use numpy's generator instead of std::mt19937 (the reference's
draws are libstdc++-specific); every check is tolerance-based, as in the
reference.
"""
import numpy as np
import pytest

from conftest import FIXTURES, fixture_path
from oracle import oracle_py as O
from paper_2501_08293_b200 import dopf

INF = float("inf")

FROZEN = {  # test_oracle.cpp:23-29
    "single_bus": (0.0405, 1e-12),
    "two_bus": (50.0 / 501.0, 1e-12),
    "three_bus_transformer": (0.3138640537987686, 1e-9),
    "four_bus_delta": (0.5020313167088988, 1e-9),
    "two_bus_delta": (0.5790045839787745, 1e-9),
}


def load(name):
    return dopf.load_model(fixture_path(name))


def rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


# ------------------------------------------------------------------ frozen objectives


@pytest.mark.parametrize("name", FIXTURES)
def test_simplex_reproduces_frozen_objective(name):
    _, ls, _ = load(name)
    ref = O.reference_solve(ls)
    assert ref["status"] == "optimal"
    want, tol = FROZEN[name]
    assert rel(ref["objective"], want) <= tol
    feas = O.check_feasibility(ls, ref["x"])
    assert feas["max_equality_violation"] <= 1e-9
    assert feas["max_bound_violation"] <= 1e-9


@pytest.mark.parametrize("name", FIXTURES)
def test_admm_oracle_within_ten_eps_of_frozen(name):
    _, _, model = load(name)
    st = dopf.Settings(eps_rel=1e-4)
    res = O.solve(model, st)
    assert res.status == dopf.CONVERGED
    assert rel(res.objective, FROZEN[name][0]) <= 10 * st.eps_rel
    assert res.max_local_infeasibility <= 1e-8   # acceptance criterion 2


def test_two_bus_objective_within_1e3_and_reconstruction_feasible():
    # test_admm.cpp:346-358, test_oracle.cpp:202-214
    _, ls, model = load("two_bus")
    res = O.solve(model, dopf.Settings(eps_rel=1e-4))
    assert res.status == dopf.CONVERGED
    assert rel(res.objective, 50.0 / 501.0) <= 1e-3
    rebuilt = O.reconstruct_centralized(model, res.x, res.z)
    feas = O.check_feasibility(ls, rebuilt)
    assert feas["max_equality_violation"] <= 1e-3
    assert feas["max_bound_violation"] <= 1e-3


def test_check_feasibility_zero_vector_exposes_rhs():
    # test_oracle.cpp:33-40
    _, ls, _ = load("two_bus")
    feas = O.check_feasibility(ls, np.zeros(ls.cols))
    assert feas["max_equality_violation"] == pytest.approx(np.abs(ls.b).max(), rel=1e-15)
    assert feas["max_bound_violation"] == pytest.approx(1.0, rel=1e-15)


# ------------------------------------------------------------------ precompute KATs


def sub(model, s=0):
    return model.subsystem(s)


def test_precompute_square_identity_pins_solution():
    m = dopf.single_sub_model(np.eye(2), [3.0, 4.0], [0, 0], [-INF, -INF], [INF, INF])
    m.precompute()
    d = sub(m)
    assert np.abs(d["P"]).max() == 0.0
    assert list(d["v"]) == [3.0, 4.0]


def test_precompute_one_row_closed_form():
    m = dopf.single_sub_model([[1.0, 0.0]], [3.0], [0, 0], [-INF, -INF], [INF, INF])
    m.precompute()
    d = sub(m)
    assert np.abs(d["P"] - np.array([[0.0, 0.0], [0.0, 1.0]])).max() <= 1e-15
    assert d["v"][0] == pytest.approx(3.0, rel=1e-15)
    assert d["v"][1] == 0.0


def random_full_row_rank(rng, m, n):
    while True:
        a = rng.standard_normal((m, n))
        if np.linalg.matrix_rank(a) == m:
            return a


def test_precompute_projector_identities_random():
    rng = np.random.default_rng(7)
    for _ in range(100):
        a = random_full_row_rank(rng, 3, 7)
        b = rng.standard_normal(3)
        m = dopf.single_sub_model(a, b, np.zeros(7), [-INF] * 7, [INF] * 7)
        m.precompute()
        d = sub(m)
        p = d["P"]
        assert np.abs(p @ p - p).max() <= 1e-9
        assert np.abs(a @ p).max() <= 1e-9
        assert np.abs(a @ d["v"] - b).max() <= 1e-9


def test_precompute_rank_deficient_raises_singular():
    m = dopf.single_sub_model([[1.0, 0, 0], [1.0, 0, 0]], [1.0, 1.0], np.zeros(3), [-INF] * 3,
                              [INF] * 3)
    with pytest.raises(dopf.SingularSubsystemError):
        m.precompute()


def test_precompute_no_rows_is_identity():
    m = dopf.single_sub_model(np.zeros((0, 2)), [], [0, 0], [-INF, -INF], [INF, INF])
    m.precompute()
    d = sub(m)
    assert np.array_equal(d["P"], np.eye(2))
    assert list(d["v"]) == [0.0, 0.0]


# ------------------------------------------------------------------ step KATs


def one_col(c, lo, hi):
    m = dopf.single_sub_model(np.zeros((0, 1)), [], [c], [lo], [hi])
    m.precompute()
    return m


@pytest.mark.parametrize("c,lo,hi,rho,want", [(0.0, 0.0, 10.0, 100.0, 5.0),   # average
                                              (0.0, 0.0, 3.0, 100.0, 3.0),    # clamp
                                              (1.0, -INF, INF, 1.0, 4.0)])    # cost shift
def test_global_update_single_copy(c, lo, hi, rho, want):
    m = one_col(c, lo, hi)
    x = O.global_update(m, [5.0], [0.0], rho)
    assert x[0] == want


def test_global_update_divides_by_copy_count():
    m = dopf.model_from_arrays([(np.zeros((0, 1)), [], [0]), (np.zeros((0, 1)), [], [0])],
                               [0.0], [-INF], [INF])
    m.precompute()
    assert m.arr("inv_copy")[0] == 0.5
    x = O.global_update(m, [0.9, 1.1], [0.0, 0.0], 100.0)
    assert x[0] == pytest.approx(1.0, rel=1e-15)


def test_local_update_fully_determined_ignores_target():
    m = dopf.single_sub_model(np.eye(2), [3.0, 4.0], [0, 0], [-INF, -INF], [INF, INF])
    m.precompute()
    z = O.local_update(m, 0, [7.0, -2.0], [1.0, 1.0], 100.0)
    assert np.abs(z - [3.0, 4.0]).max() <= 1e-12


def test_local_update_pins_constrained_frees_other():
    m = dopf.single_sub_model([[1.0, 0.0]], [3.0], [0, 0], [-INF, -INF], [INF, INF])
    m.precompute()
    z = O.local_update(m, 0, [2.0, 4.0], [0.0, 0.0], 1.0)
    assert z[0] == pytest.approx(3.0, rel=1e-15)
    assert z[1] == pytest.approx(4.0, rel=1e-15)


def kkt_minimizer(a, b, d, rho):
    m, n = a.shape
    k = np.zeros((n + m, n + m))
    k[:n, :n] = rho * np.eye(n)
    k[:n, n:] = a.T
    k[n:, :n] = a
    return np.linalg.solve(k, np.concatenate([-d, b]))[:n]


@pytest.mark.parametrize("seed,trials", [(99, 50), (424242, 200)])  # test_admm :189, criterion 4
def test_local_update_matches_dense_kkt(seed, trials):
    rng = np.random.default_rng(seed)
    for _ in range(trials):
        mm = int(rng.integers(1, 11))
        n = mm + int(rng.integers(0, 11))
        rho = float(rng.uniform(0.5, 200.0))
        a = random_full_row_rank(rng, mm, n)
        b = rng.standard_normal(mm)
        model = dopf.single_sub_model(a, b, np.zeros(n), [-INF] * n, [INF] * n)
        model.precompute()
        xg = rng.normal(0, 2.0, n)
        lam = rng.normal(0, 5.0, n)
        mine = O.local_update(model, 0, xg, lam, rho)
        want = kkt_minimizer(a, b, -rho * xg - lam, rho)
        assert np.abs(mine - want).max() <= 1e-8
        assert np.abs(a @ mine - b).max() <= 1e-8


def test_dual_update_consensus_keeps_gap_moves():
    m = dopf.single_sub_model([[1.0, 1.0]], [1.0], [0, 0], [-INF, -INF], [INF, INF])
    m.precompute()
    xg = np.array([0.25, 0.75])
    lam = O.dual_update(m, 0, xg, xg, [3.0, -1.0], 100.0)
    assert list(lam) == [3.0, -1.0]
    zs = xg.copy()
    zs[0] -= 0.01
    lam = O.dual_update(m, 0, xg, zs, lam, 100.0)
    assert lam[0] == pytest.approx(4.0, rel=1e-15)
    assert lam[1] == -1.0


def test_dual_update_two_bus_first_iteration_by_hand():
    _, _, m = load("two_bus")
    m.precompute()
    rho = 100.0
    z0 = m.arr("z0")
    x = O.global_update(m, z0, np.zeros_like(z0), rho)
    zo = m.z_offsets
    ns = zo[1] - zo[0]
    zs = O.local_update(m, 0, x, np.zeros(ns), rho)
    lam = O.dual_update(m, 0, x, zs, np.zeros(ns), rho)
    l2g = m.arr("l2g")[zo[0]:zo[1]]
    for j in range(ns):
        assert lam[j] == pytest.approx(rho * (x[l2g[j]] - zs[j]), rel=1e-12)


def test_residuals_vanish_at_consensus():
    m = dopf.single_sub_model(np.zeros((0, 2)), [], [0, 0], [-INF, -INF], [INF, INF])
    m.precompute()
    x = np.array([1.0, 2.0])
    pres, dres, ep, ed = O.residuals(m, x, x, x, np.zeros(2), 100.0, 1e-3)
    assert pres == 0.0 and dres == 0.0 and pres <= ep and dres <= ed


def test_residuals_scalar_formulas():
    m = dopf.single_sub_model(np.zeros((0, 1)), [], [0.0], [-INF], [INF])
    m.precompute()
    pres, dres, ep, ed = O.residuals(m, [1.3], [1.0], [1.0], [10.0], 100.0, 1e-3)
    assert pres == pytest.approx(0.3, rel=1e-15)
    assert dres == 0.0
    assert ep == pytest.approx(1e-3 * 1.3, rel=1e-15)
    assert ed == pytest.approx(1e-3 * 10.0, rel=1e-15)


def test_initialize_voltage_rule_then_midpoint_then_zero():
    _, ls, m = load("two_bus")
    x0 = m.arr("x0")
    assert x0[ls.column("w:b1:1")] == 1.0
    assert x0[ls.column("p_gen:g1:1")] == 1.0
    assert x0[ls.column("q_gen:g1:1")] == 0.0
    assert x0[ls.column("p_load:d1:1")] == 0.0
    z0, l2g = m.arr("z0"), m.arr("l2g")
    assert np.array_equal(z0, x0[l2g])


# ------------------------------------------------------------------ solve KATs


def test_solve_square_model_converges_to_unique_point():
    a = np.array([[2.0, 1.0], [1.0, 3.0]])
    sol = np.array([0.4, 0.7])
    m = dopf.single_sub_model(a, a @ sol, [1.0, 0.0], [-10, -10], [10, 10])
    res = O.solve(m, dopf.Settings(eps_rel=1e-8, max_iter=100))
    assert res.status == dopf.CONVERGED
    assert np.abs(res.x - sol).max() <= 1e-10
    assert res.trace[-1, 1] <= res.trace[-1, 3] and res.trace[-1, 2] <= res.trace[-1, 4]


def test_solve_iteration_cap_is_a_status():
    _, _, m = load("two_bus")
    res = O.solve(m, dopf.Settings(eps_rel=1e-12, max_iter=10))
    assert res.status == dopf.ITERATION_LIMIT
    assert res.iterations == 10 and res.trace.shape == (10, 6)
    lo, hi = m.arr("x_lo"), m.arr("x_hi")
    assert np.all(res.x >= lo) and np.all(res.x <= hi)


@pytest.mark.parametrize("name", ["three_bus_transformer", "four_bus_delta"])
def test_solve_bitwise_across_worker_counts(name):
    # test_admm.cpp:376-394, acceptance criterion 6
    _, _, m = load(name)
    runs = [O.solve(m, dopf.Settings(eps_rel=1e-4, workers=w)) for w in (1, 2, 4)]
    for r in runs[1:]:
        assert np.array_equal(r.trace, runs[0].trace)
        assert np.array_equal(r.x, runs[0].x)


def test_solve_rejects_invalid_settings():
    m = dopf.single_sub_model(np.eye(1), [1.0], [0.0], [-INF], [INF])
    for bad in (dopf.Settings(rho=0.0), dopf.Settings(eps_rel=0.0), dopf.Settings(max_iter=0)):
        with pytest.raises(ValueError):
            O.solve(m, bad)


def test_trace_matches_independent_recomputation():
    # acceptance criterion 5: termination formulas from snapshots, <= 1e-12
    _, _, m = load("four_bus_delta")
    st = dopf.Settings(eps_rel=1e-4)
    samples = [1, 2, 3, 7, 20, 50]
    res = O.solve(m, st, snap_iters=samples)
    rho, eps = st.rho, st.eps_rel
    for t in samples:
        if t > res.iterations:
            continue
        s = res.snapshots[t]
        x, z, zp, lam = s["x"], s["z"], s["z_prev"], s["lambda"]
        bx = x[m.arr("l2g")]
        pres = np.sqrt(np.sum((bx - z) ** 2))
        dres = rho * np.sqrt(np.sum((z - zp) ** 2))
        ep = eps * max(np.linalg.norm(bx), np.linalg.norm(z))
        ed = eps * np.linalg.norm(lam)
        row = res.trace[t - 1]
        for got, want in zip(row[1:5], (pres, dres, ep, ed)):
            assert abs(got - want) <= 1e-12 * max(1.0, abs(want))


def test_iterations_monotone_in_tolerance():
    # acceptance criterion 9
    _, _, m = load("three_bus_transformer")
    its = [O.solve(m, dopf.Settings(eps_rel=e)).iterations for e in (1e-2, 1e-3, 1e-4)]
    assert its[0] <= its[1] <= its[2]
