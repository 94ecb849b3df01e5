"""Host front-end (the path's input producer) against the reference's pinned
structure: LP dimensions (proj/tests/test_lp_builder.cpp:50, 359), component
order and pre-reduction subsystem shapes (checked
against test_decompose.cpp:132-147 and test_cli.cpp:93), and the synthetic
feeders' structural counts against the paper's Table II."""
import numpy as np
import pytest

from conftest import fixture_path
from paper_2501_08293_b200 import dopf

APPENDIX_A = {
    "single_bus": (3, 2, ["bus:sub"], [(2, 3)], 3),
    "two_bus": (12, 11, ["leaf:b1+ln1", "bus:sub"], [(9, 10), (2, 4)], 14),
    "two_bus_delta": (36, 33, ["leaf:b1+ln1", "bus:sub"], [(27, 30), (6, 12)], 42),
    "three_bus_transformer": (34, 32, ["bus:b1", "leaf:b2+xf1", "leaf:sub+ln1"],
                              [(4, 10), (18, 20), (10, 16)], 46),
    "four_bus_delta": (68, 65, ["bus:b1", "leaf:b2+ln2", "leaf:b3+ln3", "leaf:sub+ln1"],
                       [(14, 24), (9, 10), (27, 30), (15, 24)], 88),
}


@pytest.mark.parametrize("name", sorted(APPENDIX_A))
def test_fixture_structure(name):
    cols, rows, comps, shapes, nz = APPENDIX_A[name]
    _, ls, m = dopf.load_model(fixture_path(name))
    assert (ls.cols, ls.rows) == (cols, rows)
    assert [m.component_id(s) for s in range(m.S)] == comps
    got = list(zip(m.rows_before_reduction().tolist(), np.diff(m.z_offsets).tolist()))
    assert got == shapes
    assert m.total_local_vars == nz


def test_two_bus_copy_counts_only_on_flows():
    # test_decompose.cpp:132-147: copy count 2 only on the line's p/q (from-to)
    _, ls, m = dopf.load_model(fixture_path("two_bus"))
    counts = m.copy_counts
    shared = [ls.var_key(j) for j in range(ls.cols) if counts[j] == 2]
    assert shared and all(k.startswith(("p_flow", "q_flow")) for k in shared)
    assert all(c in (1, 2) for c in counts)


@pytest.mark.parametrize("shape,seed,counts,S,n", [
    ("ieee13", 13, (29, 28, 7), 50, 454),
    ("ieee123", 123, (147, 146, 43), 250, 1834),
    ("ieee8500", 8500, (11932, 14291, 1222), 25001, 87285),
])
def test_synthetic_feeders_match_paper_table2(shape, seed, counts, S, n):
    f = dopf.synthetic_feeder(shape, seed)
    c = f.counts()
    assert (c["buses"], c["lines"], c["leaves"]) == counts
    assert not dopf.has_errors(dopf.validate_feeder(f))
    _, ls, m = dopf.load_model(f, workers=4)
    assert m.S == S and ls.cols == n


def test_synthetic_feeder_is_deterministic():
    a = dopf.synthetic_feeder("ieee123", 123).serialize()
    b = dopf.synthetic_feeder("ieee123", 123).serialize()
    c = dopf.synthetic_feeder("ieee123", 124).serialize()
    assert a == b and a != c


def test_scenario_scaling_keeps_structure():
    base = dopf.synthetic_feeder("ieee123", 123)
    _, _, m0 = dopf.load_model(base)
    for k in range(3):
        f = dopf.scale_loads(base, 4096 + k)
        _, _, m = dopf.load_model(f)
        assert m.S == m0.S and np.array_equal(m.z_offsets, m0.z_offsets)
        assert np.array_equal(m.arr("l2g"), m0.arr("l2g"))


def test_parse_roundtrip_and_errors():
    f = dopf.parse_feeder_file(fixture_path("four_bus_delta"))
    g = dopf.parse_feeder(f.serialize())
    assert g.serialize() == f.serialize()
    with pytest.raises(dopf.ParseError):
        dopf.parse_feeder('{"buses": [], "unknown_key": 1}')


def test_trace_csv_format():
    # admm.cpp:246-252: header + precision 17
    tr = np.array([[1, 0.5, 0.25, 1e-3, 2e-3, 0.1]])
    text = dopf.write_trace_csv(tr)
    lines = text.strip().splitlines()
    assert lines[0] == "t,pres,dres,eps_prim,eps_dual,objective"
    assert lines[1].startswith("1,0.5,0.25,")
