"""The reference's decomposition tests (proj/tests/test_decompose.cpp)
restated against the product's host front-end (csrc/host/decompose.cpp):
component graph, partition, row_reduce (pivot normalisation, infeasibility,
row space, sub-tolerance noise, the named failing subsystem), feasibility
transport of the centralized LP optimum, and the random-feeder pipeline
property (test_decompose.cpp:296-331) over 20 radial feeders."""
import json

import numpy as np
import pytest

from conftest import fixture_path
from feeder_gen import random_feeder
from oracle import oracle_py as O
from paper_2501_08293_b200 import dopf

FIXTURES = ["single_bus", "two_bus", "two_bus_delta", "three_bus_transformer", "four_bus_delta"]


def bus(i, ph=(1,)):
    return {"id": i, "phases": list(ph), "w_lo": [0.81] * len(ph), "w_hi": [1.21] * len(ph)}


def line(i, a, b):
    return {"id": i, "from_bus": a, "to_bus": b, "phases": [1], "r": [[0.01]], "x": [[0.02]]}


def path_feeder(n):
    return {"base": 1.0, "buses": [bus(f"b{i}") for i in range(n)],
            "generators": [{"id": "g0", "bus": "b0", "phases": [1], "p_lo": [0.0], "p_hi": [2.0],
                            "q_lo": [-2.0], "q_hi": [2.0]}],
            "lines": [line(f"e{i}", f"b{i}", f"b{i + 1}") for i in range(n - 1)], "loads": []}


def model_of(d, reduce=True):
    f = dopf.parse_feeder(json.dumps(d) if isinstance(d, dict) else d)
    ls = dopf.assemble_centralized(f)
    m = dopf.partition(ls, f)
    if reduce:
        m.reduce()
    return f, ls, m


def comps(m):
    return [m.component_id(s) for s in range(m.S)]


def test_component_graph_path_merges_both_ends():
    _, _, m = model_of(path_feeder(3), reduce=False)
    c = comps(m)
    assert len(c) == 3  # |buses| + |lines| - |leaves| = 3 + 2 - 2
    assert sum(x.startswith("leaf:") for x in c) == 2
    assert sum(x.startswith("bus:") for x in c) == 1
    assert not any(x.startswith("line:") for x in c)


def test_component_graph_star_with_four_leaves():
    d = path_feeder(1)
    for i in range(1, 5):
        d["buses"].append(bus(f"leaf{i}"))
        d["lines"].append(line(f"e{i}", "b0", f"leaf{i}"))
    _, _, m = model_of(d, reduce=False)
    assert len(comps(m)) == 5  # 5 + 4 - 4


@pytest.mark.parametrize("name", FIXTURES)
def test_component_members_partition_buses_and_lines(name):
    f = dopf.parse_feeder_file(fixture_path(name))
    d = json.loads(f.serialize())
    _, _, m = model_of(d, reduce=False)
    buses, lines = [], []
    for cid in comps(m):
        kind, rest = cid.split(":", 1)
        if kind == "leaf":
            b, ln = rest.split("+", 1)
            buses.append(b)
            lines.append(ln)
        elif kind == "bus":
            buses.append(rest)
        else:
            lines.append(rest)
    assert sorted(buses) == sorted(b["id"] for b in d["buses"]) and len(set(buses)) == len(buses)
    assert sorted(lines) == sorted(x["id"] for x in d["lines"]) and len(set(lines)) == len(lines)


def test_partition_single_component_keeps_dense_system():
    d = path_feeder(1)
    d["buses"][0].update(g_sh=[0.05], b_sh=[0.02])
    _, ls, m = model_of(d, reduce=False)
    assert m.S == 1
    sub = m.subsystem(0)
    assert sub["A"].shape == (ls.rows, ls.cols)
    assert list(sub["local_to_global"]) == [0, 1, 2]  # identity consensus map
    assert np.abs(ls.dense() - sub["A"]).max() == 0.0


def test_partition_two_bus_shares_only_from_side_flows():
    _, ls, m = model_of(dopf.parse_feeder_file(fixture_path("two_bus")).serialize(), reduce=False)
    assert m.S == 2
    keys = ls.var_table()
    for col, cnt in enumerate(m.copy_counts):
        assert cnt == (2 if keys[col] in ("p_flow:ln1:1:ft", "q_flow:ln1:1:ft") else 1), keys[col]


@pytest.mark.parametrize("name", FIXTURES)
def test_partition_copy_counts_and_offsets(name):
    _, ls, m = model_of(dopf.parse_feeder_file(fixture_path(name)).serialize(), reduce=False)
    assert (m.copy_counts >= 1).all()
    total = rows = 0
    for s in range(m.S):
        l2g = m.subsystem(s)["local_to_global"]
        total += len(l2g)
        assert (np.diff(l2g) > 0).all()  # strictly ascending -> duplicate free
    rows = int(m.rows_before_reduction().sum())
    assert m.total_local_vars == total
    assert rows == ls.rows  # every centralized row lands in exactly one subsystem


def test_partition_voltage_column_without_rows_gets_a_home():
    _, _, m = model_of(path_feeder(1), reduce=False)
    assert (m.copy_counts == 1).all()


def reduced(a, b, tol=1e-9):
    a = np.asarray(a, dtype=np.float64)
    m = dopf.single_sub_model(a, b, np.zeros(a.shape[1]), [-np.inf] * a.shape[1], [np.inf] * a.shape[1])
    m.reduce(tol)
    s = m.subsystem(0)
    return s["A"], s["b"]


def test_row_reduce_drops_duplicate_and_normalizes():
    a2, b2 = reduced([[1, 0], [2, 0]], [3, 6])
    assert a2.shape == (1, 2) and a2[0, 0] == 1.0 and a2[0, 1] == 0.0
    assert b2[0] == pytest.approx(3.0, rel=1e-15)


def test_row_reduce_contradictory_rows_infeasible():
    with pytest.raises(dopf.InfeasibleSubsystemError):
        reduced([[1, 0], [1, 0]], [3, 4])


def test_row_reduce_keeps_row_space_of_known_rank_system():
    rng = np.random.default_rng(20240817)
    g, mix = rng.normal(size=(3, 8)), rng.normal(size=(5, 3))
    a = mix @ g
    b = a @ rng.normal(size=8)
    a2, b2 = reduced(a, b)
    assert a2.shape[0] == 3
    aug = np.hstack([a2, b2[:, None]])
    for i in range(5):
        row = np.append(a[i], b[i])
        coef, *_ = np.linalg.lstsq(aug.T, row, rcond=None)
        assert np.linalg.norm(aug.T @ coef - row) <= 1e-9


def test_row_reduce_sub_tolerance_noise_is_zero():
    a2, _ = reduced([[1, 0], [1, 1e-12]], [3, 3])
    assert a2.shape[0] == 1


def test_row_reduce_first_strict_maximum_pivot():
    # equal magnitudes everywhere: the first in row-major scan order is the pivot
    a2, b2 = reduced([[1, -1, 1], [-1, 1, 1]], [2, 0])
    assert a2.shape[0] == 2
    assert list(a2[0]) == [1.0, -1.0, 1.0] and b2[0] == 2.0  # row 0 kept as is (pivot (0,0) = 1)
    assert list(a2[1]) == [0.0, 0.0, 1.0] and b2[1] == 1.0   # (-1,1,1)+(1,-1,1) = (0,0,2) / 2


def test_reduce_subsystems_names_the_offending_subsystem():
    _, _, m = model_of(dopf.parse_feeder_file(fixture_path("two_bus")).serialize(), reduce=False)
    subs = [m.subsystem(s) for s in range(m.S)]
    a0, b0 = subs[0]["A"], subs[0]["b"]
    subs[0]["A"] = np.vstack([a0, a0[:1]])
    subs[0]["b"] = np.append(b0, b0[0] + 1.0)  # a contradiction
    v = m.view()
    n = v.n
    bad = dopf.model_from_arrays([(s["A"], s["b"], list(s["local_to_global"])) for s in subs],
                                 m.arr("c"), m.arr("x_lo"), m.arr("x_hi"))
    assert n == bad.global_cols
    with pytest.raises(dopf.InfeasibleSubsystemError) as e:
        bad.reduce()
    assert e.value.subsystem_id == bad.component_id(0)


@pytest.mark.parametrize("name", FIXTURES)
def test_feasibility_transport(name):
    _, ls, pre = model_of(dopf.parse_feeder_file(fixture_path(name)).serialize(), reduce=False)
    lp = O.reference_solve(ls)
    assert lp["status"] == "optimal"
    for s in range(pre.S):
        sub = pre.subsystem(s)
        if sub["A"].shape[0]:
            assert np.abs(sub["A"] @ lp["x"][sub["local_to_global"]] - sub["b"]).max() <= 1e-9
    _, _, post = model_of(dopf.parse_feeder_file(fixture_path(name)).serialize())
    rows = 0
    for s in range(post.S):
        sub = post.subsystem(s)
        rows += sub["A"].shape[0]
        if sub["A"].shape[0]:
            assert np.abs(sub["A"] @ lp["x"][sub["local_to_global"]] - sub["b"]).max() <= 1e-9
    assert rows <= ls.rows


@pytest.mark.parametrize("seed", range(100, 120))
def test_random_feeders_decompose_cleanly(seed):
    f = dopf.parse_feeder(random_feeder(seed))
    assert not dopf.has_errors(dopf.validate_feeder(f))
    ls = dopf.assemble_centralized(f)
    m = dopf.partition(ls, f)
    assert int(m.rows_before_reduction().sum()) == ls.rows
    assert (m.copy_counts >= 1).all()
    try:
        m.reduce(1e-9, 2)
    except dopf.InfeasibleSubsystemError:
        return  # legitimate: sampled data can pin one voltage twice; detection is the contract
    m.precompute()  # independent rows only: every factorization goes through
    lp = O.reference_solve(ls)
    if lp["status"] == "optimal":
        for s in range(m.S):
            sub = m.subsystem(s)
            if sub["A"].shape[0]:
                assert np.abs(sub["A"] @ lp["x"][sub["local_to_global"]] - sub["b"]).max() <= 1e-9
