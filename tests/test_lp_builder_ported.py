"""The reference's LP-builder tests (proj/tests/test_lp_builder.cpp), restated
against the product's host front-end through its public API, plus a
differential pin: the whole centralized LP of every fixture, the synthetic
IEEE-13/123 shapes and 25 random radial feeders (test_util.hpp:77-172 ranges)
equals, bit for bit, a literal restatement of the reference builder
(oracle/lp_oracle.py: the O(bus x (lines + loads + gens)) power balance of
lp_builder.cpp:135-172, which the product rebuilds with incidence lists).
A silent coefficient-order change in the input producer fails here even
though GPU-vs-oracle parity (both fed by it) would not notice."""
import json
import math

import numpy as np
import pytest

from conftest import fixture_path
from feeder_gen import random_feeder
from oracle import lp_oracle as LO
from paper_2501_08293_b200 import dopf

FIXTURES = ["single_bus", "two_bus", "two_bus_delta", "three_bus_transformer", "four_bus_delta"]
SQ3 = math.sqrt(3.0)

ONE_BUS = """{"base": 1.0,
  "buses": [{"id": "sub", "phases": [1], "w_lo": [%s], "w_hi": [%s]%s}],
  "generators": [{"id": "g1", "bus": "sub", "phases": [1],
                  "p_lo": [0.0], "p_hi": [1.0], "q_lo": [-1.0], "q_hi": [1.0]}],
  "lines": [], "loads": []}"""


def lp_of(src):
    f = src if isinstance(src, dopf.Feeder) else (
        dopf.parse_feeder(src) if src.lstrip().startswith("{") else dopf.parse_feeder_file(fixture_path(src)))
    return f, dopf.assemble_centralized(f)


def rows_of(ls):
    """[(tag, {column key: coeff}, rhs)] in row order."""
    keys = ls.var_table()
    rp, ci, va, b = ls.row_ptr, ls.col_idx, ls.values, ls.b
    return [(ls.row_tag(i), {keys[c]: v for c, v in zip(ci[rp[i]:rp[i + 1]], va[rp[i]:rp[i + 1]])}, b[i])
            for i in range(ls.rows)]


def rows_with(rows, owner_tag):
    return [r for r in rows if r[0] == owner_tag]


# ----------------------------------------------------------- index_variables


def test_index_variables_one_bus_one_generator():
    _, ls = lp_of(ONE_BUS % ("1.0", "1.0", ""))
    assert ls.var_table() == ["p_gen:g1:1", "q_gen:g1:1", "w:sub:1"]


def test_index_variables_two_bus_blocks():
    # generator p,q (2) + voltages (2) + load columns (4) + both flow directions (4)
    _, ls = lp_of("two_bus")
    t = ls.var_table()
    assert len(t) == 12
    assert t[0].startswith("p_gen:") and t[2] == "w:b1:1" and t[3] == "w:sub:1"  # buses by id
    assert t[4].startswith("p_bus_load:") and t[8] == "p_flow:ln1:1:ft" and t[10] == "p_flow:ln1:1:tf"


@pytest.mark.parametrize("name", FIXTURES)
def test_index_variables_deterministic_and_collision_free(name):
    a = lp_of(name)[1].var_table()
    assert a == lp_of(name)[1].var_table()
    assert len(set(a)) == len(a)


# ----------------------------------------------------------- power balance


def test_power_balance_isolated_generating_bus():
    rows = rows_of(lp_of(ONE_BUS % ("0.81", "1.21", ""))[1])
    assert len(rows) == 2
    tag, p, rhs = rows[0]
    assert tag == "bus:sub:balance_p" and p == {"p_gen:g1:1": -1.0} and rhs == 0.0


def test_power_balance_signs():
    doc = """{"base": 1.0,
      "buses": [{"id": "a", "phases": [1], "w_lo": [0.81], "w_hi": [1.21], "g_sh": [0.01], "b_sh": [0.02]},
                {"id": "b", "phases": [1], "w_lo": [0.81], "w_hi": [1.21]}],
      "generators": [{"id": "g1", "bus": "a", "phases": [1], "p_lo": [0.0], "p_hi": [1.0],
                      "q_lo": [-1.0], "q_hi": [1.0]}],
      "lines": [{"id": "e1", "from_bus": "a", "to_bus": "b", "phases": [1], "r": [[0.01]], "x": [[0.02]]}],
      "loads": [{"id": "d1", "bus": "a", "connection": "wye", "phases": [1], "a": [0.1], "b": [0.05],
                 "alpha": [0.0], "beta": [0.0]}]}"""
    rows = rows_of(lp_of(doc)[1])
    (_, p, rhs), = rows_with(rows, "bus:a:balance_p")
    assert p["p_flow:e1:1:ft"] == 1.0 and p["p_bus_load:d1:1"] == 1.0
    assert p["w:a:1"] == 0.01 and p["p_gen:g1:1"] == -1.0 and rhs == 0.0
    (_, q, _), = rows_with(rows, "bus:a:balance_q")
    assert q["w:a:1"] == -0.02
    (_, pb, _), = rows_with(rows, "bus:b:balance_p")
    assert "p_flow:e1:1:tf" in pb  # the far end sees the reverse-direction flow


def test_power_balance_two_bus_has_four_rows():
    rows = rows_of(lp_of("two_bus")[1])
    assert sum(1 for r in rows if ":balance_" in r[0]) == 4


# ----------------------------------------------------------- load model


def two_bus_doc(**load):
    d = json.loads(lp_of("two_bus")[0].serialize())
    d["loads"][0].update(load)
    return json.dumps(d)


def test_load_model_constant_power_wye():
    rows = rows_of(lp_of(two_bus_doc(alpha=[0.0], beta=[0.0]))[1])
    assert sum(1 for r in rows if r[0].endswith(("load_p", "load_q", "load_link"))) == 4
    (_, d, rhs), = rows_with(rows, "bus:b1:load_p")
    assert d == {"p_load:d1:1": 1.0}  # alpha = 0 removes the voltage coupling
    assert rhs == pytest.approx(0.1, rel=1e-15)
    links = rows_with(rows, "bus:b1:load_link")
    assert len(links) == 2
    assert links[0][1] == {"p_bus_load:d1:1": 1.0, "p_load:d1:1": -1.0}


def test_load_model_voltage_coupling_wye_and_delta():
    rows = rows_of(lp_of(two_bus_doc(alpha=[1.0]))[1])
    (_, d, rhs), = rows_with(rows, "bus:b1:load_p")
    assert d["w:b1:1"] == pytest.approx(-0.05, rel=1e-15)  # -a alpha / 2
    assert rhs == pytest.approx(0.05, rel=1e-15)            # a (1 - alpha / 2)
    grows = rows_of(lp_of("two_bus_delta")[1])
    gd = rows_with(grows, "bus:b1:load_p")
    assert len(gd) == 3
    assert gd[0][1]["w:b1:1"] == pytest.approx(-0.21, rel=1e-12)  # delta: 3w, a = 0.07, alpha = 2


def test_load_model_delta_coupling_rows_as_printed():
    f, ls = lp_of("two_bus_delta")
    links = rows_with(rows_of(ls), "bus:b1:load_link")
    assert len(links) == 6
    s = links[0][1]
    assert len(s) == 6 and links[0][2] == 0.0
    for ph in (1, 2, 3):
        assert s[f"p_bus_load:d1:{ph}"] == 1.0 and s[f"p_load:d1:{ph}"] == -1.0
    r = links[2][1]  # 3/2 pb2 - sqrt3/2 qb2 - pd2 - 1/2 pd1 + sqrt3/2 qd1 = 0
    assert r["p_bus_load:d1:2"] == pytest.approx(1.5, rel=1e-15)
    assert r["q_bus_load:d1:2"] == pytest.approx(-SQ3 / 2, rel=1e-15)
    assert r["p_load:d1:2"] == -1.0 and r["p_load:d1:1"] == -0.5
    assert r["q_load:d1:1"] == pytest.approx(SQ3 / 2, rel=1e-15) and links[2][2] == 0.0
    ld = json.loads(f.serialize())["loads"][0]
    assert sum(ld["a"]) == pytest.approx(0.21, rel=1e-15)
    assert sum(ld["b"]) == pytest.approx(0.075, rel=1e-15)


# ----------------------------------------------------------- M matrices


def test_m_matrices_single_phase():
    mp, mq = dopf.line_m_matrices([1], [[0.01]], [[0.02]])
    assert mp[0, 0] == pytest.approx(-0.02, rel=1e-15) and mq[0, 0] == pytest.approx(-0.04, rel=1e-15)


def test_m_matrices_zero_mutual():
    mp, mq = dopf.line_m_matrices([1, 2, 3], np.eye(3) * 0.01, np.eye(3) * 0.02)
    assert np.abs(mp + 0.02 * np.eye(3)).max() == 0.0
    assert np.abs(mq + 0.04 * np.eye(3)).max() == 0.0


def test_m_matrices_sqrt3_pattern():
    r = np.array([[0.01, 0.003, 0.002], [0.003, 0.011, 0.004], [0.002, 0.004, 0.012]])
    x = np.array([[0.02, 0.004, 0.005], [0.004, 0.021, 0.006], [0.005, 0.006, 0.022]])
    mp, mq = dopf.line_m_matrices([1, 2, 3], r, x)
    assert mp[0, 1] == pytest.approx(0.003 - SQ3 * 0.004, rel=1e-12)
    R = lambda i, j: r[i - 1, j - 1]  # noqa: E731
    X = lambda i, j: x[i - 1, j - 1]  # noqa: E731
    emp = [[-2 * R(1, 1), R(1, 2) - SQ3 * X(1, 2), R(1, 3) + SQ3 * X(1, 3)],
           [R(2, 1) + SQ3 * X(2, 1), -2 * R(2, 2), R(2, 3) - SQ3 * X(2, 3)],
           [R(3, 1) - SQ3 * X(3, 1), R(3, 2) + SQ3 * X(3, 2), -2 * R(3, 3)]]
    emq = [[-2 * X(1, 1), X(1, 2) + SQ3 * R(1, 2), X(1, 3) - SQ3 * R(1, 3)],
           [X(2, 1) - SQ3 * R(2, 1), -2 * X(2, 2), X(2, 3) + SQ3 * R(2, 3)],
           [X(3, 1) + SQ3 * R(3, 1), X(3, 2) - SQ3 * R(3, 2), -2 * X(3, 3)]]
    np.testing.assert_allclose(mp, emp, rtol=1e-15)
    np.testing.assert_allclose(mq, emq, rtol=1e-15)


def test_m_matrices_two_phase_subset():
    mp, mq = dopf.line_m_matrices([1, 3], [[0.01, 0.003], [0.003, 0.012]], [[0.02, 0.005], [0.005, 0.022]])
    assert mp[0, 1] == pytest.approx(0.003 + SQ3 * 0.005, rel=1e-12)  # (1,3): r + sqrt3 x
    assert mp[1, 0] == pytest.approx(0.003 - SQ3 * 0.005, rel=1e-12)  # (3,1): r - sqrt3 x
    assert mq[0, 1] == pytest.approx(0.005 - SQ3 * 0.003, rel=1e-12)
    assert mq[1, 0] == pytest.approx(0.005 + SQ3 * 0.003, rel=1e-12)


# ----------------------------------------------------------- flow equations


def test_flow_equations_shunt_free_single_phase():
    rows = [r for r in rows_of(lp_of("two_bus")[1]) if r[0].startswith("line:")]
    assert len(rows) == 3
    assert rows[0][1] == {"p_flow:ln1:1:ft": 1.0, "p_flow:ln1:1:tf": 1.0} and rows[0][2] == 0.0
    tag, d, _ = rows[2]
    assert tag == "line:ln1:drop"
    assert d["w:sub:1"] == 1.0 and d["w:b1:1"] == -1.0
    assert d["p_flow:ln1:1:ft"] == pytest.approx(-0.02, rel=1e-15)
    assert d["q_flow:ln1:1:ft"] == pytest.approx(-0.04, rel=1e-15)


def test_flow_equations_line_shunts_and_tap():
    rows = [r for r in rows_of(lp_of("three_bus_transformer")[1]) if r[0].startswith("line:")]
    assert len(rows) == 12
    drops = rows_with(rows, "line:xf1:drop")
    assert len(drops) == 2
    assert drops[0][1]["w:b1:1"] == 1.0
    assert drops[0][1]["w:b2:1"] == pytest.approx(-1.0404, rel=1e-15)
    g = rows_of(lp_of("two_bus_delta")[1])
    losses = rows_with(g, "line:ln1:loss_p")
    assert len(losses) == 3
    assert losses[0][1]["w:sub:1"] == pytest.approx(-0.0015, rel=1e-15)
    assert losses[0][1]["w:b1:1"] == pytest.approx(-0.0015, rel=1e-15)
    assert rows_with(g, "line:ln1:loss_q")[0][1]["w:sub:1"] == pytest.approx(0.005, rel=1e-15)


# ----------------------------------------------------------- assemble_centralized


def test_assemble_one_bus_degenerate():
    _, ls = lp_of(ONE_BUS % ("0.81", "1.21", ""))
    assert (ls.rows, ls.cols) == (2, 3)
    assert list(ls.c) == [1.0, 0.0, 0.0]
    assert ls.x_lo[2] == 0.81 and ls.x_hi[2] == 1.21


def test_assemble_two_bus_hand_count():
    assert lp_of("two_bus")[1].rows == 11  # 4 balance + 4 load + 3 flow


def test_assemble_cost_one_exactly_on_real_generation():
    _, ls = lp_of("four_bus_delta")
    for j, k in enumerate(ls.var_table()):
        assert ls.c[j] == (1.0 if k.startswith("p_gen:") else 0.0)


def test_assemble_bounds():
    _, ls = lp_of("two_bus")
    for j, k in enumerate(ls.var_table()):
        kind = k.split(":")[0]
        if kind in ("p_bus_load", "q_bus_load", "p_load", "q_load"):
            assert ls.x_lo[j] == -np.inf and ls.x_hi[j] == np.inf
        if kind == "p_flow":  # both directions share the printed interval
            assert ls.x_lo[j] == -2.0 and ls.x_hi[j] == 2.0


@pytest.mark.parametrize("name", FIXTURES)
def test_no_orphan_columns_and_row_tags_cover_components(name):
    f, ls = lp_of(name)
    a = ls.dense()
    ref = (a != 0).any(axis=0)
    assert all(ref[j] or (np.isfinite(ls.x_lo[j]) and np.isfinite(ls.x_hi[j])) for j in range(ls.cols))
    d = json.loads(f.serialize())
    tags = [ls.row_tag(i) for i in range(ls.rows)]
    buses = {t.split(":")[1] for t in tags if t.startswith("bus:")}
    lines = {t.split(":")[1] for t in tags if t.startswith("line:")}
    assert buses == {b["id"] for b in d["buses"]}
    assert lines == {ln["id"] for ln in d["lines"]}


# ----------------------------------------------------------- differential pin


def assert_lp_equals_restatement(f):
    ref = LO.assemble_centralized(json.loads(f.serialize()))
    ls = dopf.assemble_centralized(f)
    assert ls.var_table() == ref["var_table"]
    assert ls.rows == len(ref["rows"])
    rp, ci, va, b = ls.row_ptr, ls.col_idx, ls.values, ls.b
    for i, (tag, coeffs, rhs) in enumerate(ref["rows"]):
        assert ls.row_tag(i) == tag, i
        got = list(zip(ci[rp[i]:rp[i + 1]].tolist(), va[rp[i]:rp[i + 1]].tolist()))
        assert len(got) == len(coeffs), (i, tag)
        for (gc, gv), (rc, rv) in zip(got, coeffs):  # bitwise, column by column
            assert gc == rc and np.float64(gv).view(np.uint64) == np.float64(rv).view(np.uint64), (i, tag, gc)
        assert np.float64(b[i]).view(np.uint64) == np.float64(rhs).view(np.uint64), (i, tag)
    for name in ("c", "x_lo", "x_hi"):
        assert np.array_equal(getattr(ls, name), np.array(ref[name])), name


@pytest.mark.parametrize("name", FIXTURES)
def test_lp_equals_reference_restatement_fixtures(name):
    assert_lp_equals_restatement(lp_of(name)[0])


@pytest.mark.parametrize("shape,seed", [("ieee13", 13), ("ieee123", 123), ("ieee13", 7)])
def test_lp_equals_reference_restatement_synthetic(shape, seed):
    assert_lp_equals_restatement(dopf.synthetic_feeder(shape, seed))


@pytest.mark.parametrize("seed", range(1, 26))
def test_lp_equals_reference_restatement_random_feeders(seed):
    f = dopf.parse_feeder(random_feeder(seed))
    assert not dopf.has_errors(dopf.validate_feeder(f))
    assert_lp_equals_restatement(f)


@pytest.mark.parametrize("seed", [901, 902, 903])
def test_lp_equals_reference_restatement_larger_random_feeders(seed):
    # 60-bus radial feeders: many lines / loads per bus scan in the O(N^2) loops
    assert_lp_equals_restatement(dopf.parse_feeder(random_feeder(seed, n_buses=60)))
