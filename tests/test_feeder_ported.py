"""The reference's feeder tests (proj/tests/test_feeder.cpp) restated against
the product's host front-end (csrc/host/feeder.cpp, json.cpp) through its
public API: strict schema parsing with the reference's error behaviour,
validation diagnostics, load coefficients, and serialize/parse round trips on
the fixtures and 25 random radial feeders (test_util.hpp:77-172 ranges)."""
import json
import math

import pytest

from conftest import fixture_path
from feeder_gen import random_feeder
from paper_2501_08293_b200 import dopf

FIXTURES = ["single_bus", "two_bus", "two_bus_delta", "three_bus_transformer", "four_bus_delta"]

MINIMAL = {"base": 1.0,
           "buses": [{"id": "sub", "phases": [1], "w_lo": [1.0], "w_hi": [1.0]}],
           "generators": [{"id": "g1", "bus": "sub", "phases": [1], "p_lo": [0.0], "p_hi": [1.0],
                           "q_lo": [-1.0], "q_hi": [1.0]}],
           "lines": [], "loads": []}


def doc(**edits):
    d = json.loads(json.dumps(MINIMAL))
    d.update(edits)
    return json.dumps(d)


def fixture_dict(name):
    return json.loads(dopf.parse_feeder_file(fixture_path(name)).serialize())


def errors(d):
    return dopf.has_errors(dopf.validate_feeder(dopf.parse_feeder(json.dumps(d))))


def test_smallest_valid_feeder():
    f = dopf.parse_feeder(doc())
    assert f.counts() == {"buses": 1, "generators": 1, "lines": 0, "loads": 0, "leaves": 0}
    assert json.loads(f.serialize())["buses"][0]["g_sh"] == [0.0]  # omitted shunts default to zero
    assert dopf.validate_feeder(f) == []


def test_load_on_missing_bus_is_named():
    d = doc(loads=[{"id": "d1", "bus": "b9", "connection": "wye", "phases": [1], "a": [0.1], "b": [0.0],
                    "alpha": [0.0], "beta": [0.0]}])
    with pytest.raises(dopf.ParseError, match="b9"):
        dopf.parse_feeder(d)


def test_unknown_key_is_named():
    d = json.loads(doc())
    d["buses"][0]["voltage"] = [1.0]
    with pytest.raises(dopf.ParseError, match="voltage"):
        dopf.parse_feeder(json.dumps(d))


def test_syntax_error_reports_byte_position():
    with pytest.raises(dopf.ParseError, match="byte"):
        dopf.parse_feeder('{"base": 1.0,,}')


@pytest.mark.parametrize("phases", [[1, 1], [4]])
def test_malformed_phase_sets(phases):
    d = json.loads(doc())
    d["buses"][0].update(phases=phases, w_lo=[1.0] * len(phases), w_hi=[1.0] * len(phases))
    with pytest.raises(dopf.ParseError):
        dopf.parse_feeder(json.dumps(d))


def test_two_bus_fixture_counts():
    f = dopf.parse_feeder_file(fixture_path("two_bus"))
    c = f.counts()
    assert (c["buses"], c["lines"], c["loads"]) == (2, 1, 1)
    assert dopf.validate_feeder(f) == []


def test_generator_on_missing_phase_is_flagged():
    d = json.loads(doc())
    d["buses"][0].update(phases=[1, 3], w_lo=[1.0, 1.0], w_hi=[1.0, 1.0], g_sh=[0.0, 0.0], b_sh=[0.0, 0.0])
    d["generators"][0].update(phases=[2])
    diags = dopf.validate_feeder(dopf.parse_feeder(json.dumps(d)))
    assert dopf.has_errors(diags) and diags[0].component == "g1"


def test_pinned_voltage_bounds_allowed():
    assert dopf.validate_feeder(dopf.parse_feeder(doc())) == []


def test_disconnected_graph_is_flagged():
    d = json.loads(doc())
    d["buses"] = [{"id": "a", "phases": [1], "w_lo": [0.81], "w_hi": [1.21]},
                  {"id": "b", "phases": [1], "w_lo": [0.81], "w_hi": [1.21]}]
    d["generators"][0]["bus"] = "a"
    diags = dopf.validate_feeder(dopf.parse_feeder(json.dumps(d)))
    assert dopf.has_errors(diags) and any("disconnected" in x.message for x in diags)


def test_partial_phase_delta_load_rejected():
    d = fixture_dict("two_bus_delta")
    ld = d["loads"][0]
    for k in ("a", "b", "alpha", "beta"):
        ld[k] = ld[k][:2]
    ld["phases"] = [1, 2]
    assert errors(d)


def test_ordered_bounds_and_positive_taps():
    d = fixture_dict("two_bus")
    d["buses"][1]["w_lo"][0] = 2.0  # above w_hi
    assert errors(d)
    d = fixture_dict("two_bus")
    d["lines"][0]["tau"][0] = 0.0
    assert errors(d)
    d = fixture_dict("two_bus")
    d["loads"][0]["alpha"][0] = -1.0
    assert errors(d)


def test_derive_load_coefficients_kinds():
    cp = dopf.derive_load_coefficients(0.1, 0.05, "constant_power")
    assert cp == {"a": 0.1, "b": 0.05, "alpha": 0.0, "beta": 0.0}
    assert dopf.derive_load_coefficients(0.1, 0.05, "constant_current")["alpha"] == 1.0
    cz = dopf.derive_load_coefficients(0.1, 0.05, "constant_impedance")
    assert cz["alpha"] == 2.0 and cz["beta"] == 2.0


def demand_at(lc, w_hat):
    return lc["a"] * lc["alpha"] / 2.0 * (w_hat - 1.0) + lc["a"]


def test_load_linearization():
    assert demand_at(dopf.derive_load_coefficients(0.1, 0.05, "constant_power"), 0.5) == pytest.approx(0.1, rel=1e-15)
    cz = dopf.derive_load_coefficients(0.1, 0.05, "constant_impedance")
    assert demand_at(cz, 1.21) == pytest.approx(0.1 * 1.21, rel=1e-15)  # exact for alpha = 2
    ci = dopf.derive_load_coefficients(0.1, 0.05, "constant_current")
    assert demand_at(ci, 1.21) == pytest.approx(0.1105, rel=1e-12)
    assert abs(demand_at(ci, 1.21) - 0.1 * math.sqrt(1.21)) < 6e-4
    for kind in dopf.LOAD_KINDS:
        assert demand_at(dopf.derive_load_coefficients(0.37, 0.11, kind), 1.0) == 0.37


@pytest.mark.parametrize("name", FIXTURES)
def test_round_trip_fixtures(name):
    f = dopf.parse_feeder_file(fixture_path(name))
    text = f.serialize()
    assert dopf.parse_feeder(text).serialize() == text
    assert json.loads(text) == fixture_dict(name)


def test_round_trip_keeps_unbounded_flow_limits():
    d = fixture_dict("two_bus")
    d["lines"][0]["p_hi"][0] = None
    d["lines"][0]["p_lo"][0] = None
    g = json.loads(dopf.parse_feeder(json.dumps(d)).serialize())
    assert g["lines"][0]["p_hi"][0] is None and g["lines"][0]["p_lo"][0] is None
    ls = dopf.assemble_centralized(dopf.parse_feeder(json.dumps(d)))
    col = ls.column("p_flow:ln1:1:ft")
    assert math.isinf(ls.x_hi[col]) and math.isinf(ls.x_lo[col])


@pytest.mark.parametrize("seed", range(1, 26))
def test_round_trip_random_feeders(seed):
    f = dopf.parse_feeder(random_feeder(seed))
    assert not dopf.has_errors(dopf.validate_feeder(f))
    text = f.serialize()
    assert dopf.parse_feeder(text).serialize() == text
    # every value survives bit for bit (shortest round-trip decimal)
    src = json.loads(random_feeder(seed))
    out = json.loads(text)
    for kind in ("buses", "lines", "loads", "generators"):
        by_id = {o["id"]: o for o in out[kind]}
        for o in src[kind]:
            for k, v in o.items():
                if k == "connection" and v == "wye" and k not in by_id[o["id"]]:
                    continue
                assert by_id[o["id"]][k] == v, (kind, o["id"], k)


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_type_invariants(name):
    d = fixture_dict(name)
    for b in d["buses"]:
        assert all(0 <= lo <= hi for lo, hi in zip(b["w_lo"], b["w_hi"]))
    ids = {b["id"] for b in d["buses"]}
    for g in d["generators"]:
        assert g["bus"] in ids
        assert all(lo <= hi for lo, hi in zip(g["p_lo"], g["p_hi"]))
        assert all(lo <= hi for lo, hi in zip(g["q_lo"], g["q_hi"]))
    for ln in d["lines"]:
        n = len(ln["phases"])
        assert all(t > 0 for t in ln["tau"])
        assert all(ln["r"][a][b] == ln["r"][b][a] and ln["x"][a][b] == ln["x"][b][a]
                   for a in range(n) for b in range(n))
    for ld in d["loads"]:
        assert all(a >= 0 for a in ld["alpha"]) and all(b >= 0 for b in ld["beta"])
        if ld.get("connection") == "delta":
            assert len(ld["phases"]) == 3


def test_collections_sorted_by_string_id():
    # parse sorts every collection by id in string order (feeder.cpp canonical order)
    d = json.loads(doc())
    d["buses"] = [{"id": i, "phases": [1], "w_lo": [0.81], "w_hi": [1.21]} for i in ("b10", "b2", "a")]
    d["generators"][0]["bus"] = "a"
    d["lines"] = [{"id": "l2", "from_bus": "a", "to_bus": "b2", "phases": [1], "r": [[0.01]], "x": [[0.02]]},
                  {"id": "l1", "from_bus": "a", "to_bus": "b10", "phases": [1], "r": [[0.01]], "x": [[0.02]]}]
    out = json.loads(dopf.parse_feeder(json.dumps(d)).serialize())
    assert [b["id"] for b in out["buses"]] == ["a", "b10", "b2"]
    assert [ln["id"] for ln in out["lines"]] == ["l1", "l2"]
