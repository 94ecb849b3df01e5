"""TEST INFRASTRUCTURE ONLY -- never imported by the product path.

Literal restatement of the reference LP builder (proj/src/lp_builder.cpp)
in plain Python, used to pin the product's host input producer
(csrc/host/lp_builder.cpp, which rebuilds the O(bus x (lines + loads +
gens)) loops of build_power_balance with per-bus incidence lists). Every
loop keeps the reference's nesting and every coefficient the reference's
expression and accumulation order, so the two must agree bit for bit:

  index_variables       lp_builder.cpp:91-116   gens, buses, loads, lines blocks
  RowBuilder            lp_builder.cpp:46-64    per-column `+=` in insertion order,
                                                emission sorted by column, exact zeros dropped
  build_power_balance   lp_builder.cpp:135-172  the O(N^2) scan over all lines / loads / gens
  build_load_model      lp_builder.cpp:174-273  wye and delta (coupling rows as printed)
  build_m_matrices      lp_builder.cpp:275-296  the +-sqrt(3) cyclic pattern
  build_flow_equations  lp_builder.cpp:298-339
  assemble_centralized  lp_builder.cpp:341-410  cost 1 on p_gen, component bounds

Input: the feeder as the product serializes it (serialize_feeder, JSON with
collections in canonical string-id order and null for infinite bounds).
"""
from __future__ import annotations

import math
from typing import Dict, List, Tuple

SQRT3 = math.sqrt(3.0)
INF = math.inf


def _bound(v, default):
    return default if v is None else float(v)


def _fkey(kind: str, owner: str, phase: int, direction: str = "ft") -> str:
    s = f"{kind}:{owner}:{phase}"
    return s + (":" + direction if kind in ("p_flow", "q_flow") else "")


def index_variables(f: dict) -> List[str]:
    table = []
    for g in f["generators"]:
        for ph in g["phases"]:
            table += [_fkey("p_gen", g["id"], ph), _fkey("q_gen", g["id"], ph)]
    for b in f["buses"]:
        for ph in b["phases"]:
            table.append(_fkey("w", b["id"], ph))
    for ld in f["loads"]:
        for ph in ld["phases"]:
            table += [_fkey(k, ld["id"], ph) for k in ("p_bus_load", "q_bus_load", "p_load", "q_load")]
    for ln in f["lines"]:
        for ph in ln["phases"]:
            table += [_fkey("p_flow", ln["id"], ph, "ft"), _fkey("q_flow", ln["id"], ph, "ft"),
                      _fkey("p_flow", ln["id"], ph, "tf"), _fkey("q_flow", ln["id"], ph, "tf")]
    return table


class _Row:
    def __init__(self, tag: str, rhs: float):
        self.tag, self.rhs, self.c = tag, rhs, {}

    def add(self, col: int, v: float):
        self.c[col] = self.c.get(col, 0.0) + v

    def finish(self) -> Tuple[str, List[Tuple[int, float]], float]:
        return self.tag, [(k, self.c[k]) for k in sorted(self.c) if self.c[k] != 0.0], self.rhs


def build_power_balance(f: dict, at: Dict[str, int]):
    rows = []
    for bus in f["buses"]:
        for pi, ph in enumerate(bus["phases"]):
            p = _Row(f"bus:{bus['id']}:balance_p", 0.0)
            q = _Row(f"bus:{bus['id']}:balance_q", 0.0)
            for ln in f["lines"]:
                if ph not in ln["phases"]:
                    continue
                if ln["from_bus"] == bus["id"]:
                    p.add(at[_fkey("p_flow", ln["id"], ph, "ft")], 1.0)
                    q.add(at[_fkey("q_flow", ln["id"], ph, "ft")], 1.0)
                if ln["to_bus"] == bus["id"]:
                    p.add(at[_fkey("p_flow", ln["id"], ph, "tf")], 1.0)
                    q.add(at[_fkey("q_flow", ln["id"], ph, "tf")], 1.0)
            for ld in f["loads"]:
                if ld["bus"] != bus["id"] or ph not in ld["phases"]:
                    continue
                p.add(at[_fkey("p_bus_load", ld["id"], ph)], 1.0)
                q.add(at[_fkey("q_bus_load", ld["id"], ph)], 1.0)
            w = at[_fkey("w", bus["id"], ph)]
            p.add(w, float(bus["g_sh"][pi]))
            q.add(w, -float(bus["b_sh"][pi]))
            for g in f["generators"]:
                if g["bus"] != bus["id"] or ph not in g["phases"]:
                    continue
                p.add(at[_fkey("p_gen", g["id"], ph)], -1.0)
                q.add(at[_fkey("q_gen", g["id"], ph)], -1.0)
            rows += [p.finish(), q.finish()]
    return rows


def build_load_model(f: dict, at: Dict[str, int]):
    rows = []
    for ld in f["loads"]:
        delta = ld.get("connection", "wye") == "delta"
        w_scale = 3.0 if delta else 1.0
        tag = f"bus:{ld['bus']}:"
        for pi, ph in enumerate(ld["phases"]):
            a, b = float(ld["a"][pi]), float(ld["b"][pi])
            al, be = float(ld["alpha"][pi]), float(ld["beta"][pi])
            w = at[_fkey("w", ld["bus"], ph)]
            r = _Row(tag + "load_p", a * (1.0 - al / 2.0))
            r.add(at[_fkey("p_load", ld["id"], ph)], 1.0)
            r.add(w, -a * al / 2.0 * w_scale)
            rows.append(r.finish())
            r = _Row(tag + "load_q", b * (1.0 - be / 2.0))
            r.add(at[_fkey("q_load", ld["id"], ph)], 1.0)
            r.add(w, -b * be / 2.0 * w_scale)
            rows.append(r.finish())
        if not delta:
            for ph in ld["phases"]:
                for pk, dk in (("p_bus_load", "p_load"), ("q_bus_load", "q_load")):
                    r = _Row(tag + "load_link", 0.0)
                    r.add(at[_fkey(pk, ld["id"], ph)], 1.0)
                    r.add(at[_fkey(dk, ld["id"], ph)], -1.0)
                    rows.append(r.finish())
            continue

        def c(kind, ph, _id=ld["id"]):
            return at[_fkey(kind, _id, ph)]
        link = tag + "load_link"
        sp, sq = _Row(link, 0.0), _Row(link, 0.0)
        for ph in (1, 2, 3):
            sp.add(c("p_bus_load", ph), 1.0)
            sp.add(c("p_load", ph), -1.0)
            sq.add(c("q_bus_load", ph), 1.0)
            sq.add(c("q_load", ph), -1.0)
        rows += [sp.finish(), sq.finish()]
        for terms in (
            [("p_bus_load", 2, 1.5), ("q_bus_load", 2, -SQRT3 / 2.0), ("p_load", 2, -1.0),
             ("p_load", 1, -0.5), ("q_load", 1, SQRT3 / 2.0)],
            [("p_bus_load", 2, SQRT3 / 2.0), ("q_bus_load", 2, 1.5), ("p_load", 1, -SQRT3 / 2.0),
             ("q_load", 1, -0.5), ("q_load", 2, -1.0)],
            [("q_bus_load", 2, SQRT3), ("p_bus_load", 3, 1.5), ("q_bus_load", 3, -SQRT3 / 2.0),
             ("p_load", 1, -0.5), ("q_load", 1, -SQRT3 / 2.0), ("p_load", 3, -1.0)],
            [("p_bus_load", 2, -SQRT3), ("p_bus_load", 3, SQRT3 / 2.0), ("q_bus_load", 3, 1.5),
             ("p_load", 1, SQRT3 / 2.0), ("q_load", 1, -0.5), ("q_load", 3, -1.0)]):
            r = _Row(link, 0.0)
            for kind, ph, v in terms:
                r.add(c(kind, ph), v)
            rows.append(r.finish())
    return rows


def build_m_matrices(phases: List[int], r, x):
    n = len(phases)
    mp = [[0.0] * n for _ in range(n)]
    mq = [[0.0] * n for _ in range(n)]
    for i in range(n):
        for j in range(n):
            rv, xv = float(r[i][j]), float(x[i][j])
            if i == j:
                mp[i][j], mq[i][j] = -2.0 * rv, -2.0 * xv
            elif phases[j] == phases[i] % 3 + 1:  # cyclic successor 1 -> 2 -> 3 -> 1
                mp[i][j], mq[i][j] = rv - SQRT3 * xv, xv + SQRT3 * rv
            else:
                mp[i][j], mq[i][j] = rv + SQRT3 * xv, xv - SQRT3 * rv
    return mp, mq


def build_flow_equations(f: dict, at: Dict[str, int]):
    rows = []
    for ln in f["lines"]:
        ph = ln["phases"]
        mp, mq = build_m_matrices(ph, ln["r"], ln["x"])
        gf, bf = [float(v) for v in ln["g_s_from"]], [float(v) for v in ln["b_s_from"]]
        gt, bt = [float(v) for v in ln["g_s_to"]], [float(v) for v in ln["b_s_to"]]
        tag = f"line:{ln['id']}:"
        for i, p in enumerate(ph):
            wf, wt = at[_fkey("w", ln["from_bus"], p)], at[_fkey("w", ln["to_bus"], p)]
            r = _Row(tag + "loss_p", 0.0)
            r.add(at[_fkey("p_flow", ln["id"], p, "ft")], 1.0)
            r.add(at[_fkey("p_flow", ln["id"], p, "tf")], 1.0)
            r.add(wf, -gf[i])
            r.add(wt, -gt[i])
            rows.append(r.finish())
            r = _Row(tag + "loss_q", 0.0)
            r.add(at[_fkey("q_flow", ln["id"], p, "ft")], 1.0)
            r.add(at[_fkey("q_flow", ln["id"], p, "tf")], 1.0)
            r.add(wf, bf[i])
            r.add(wt, bt[i])
            rows.append(r.finish())
            r = _Row(tag + "drop", 0.0)
            r.add(wf, 1.0)
            r.add(wt, -float(ln["tau"][i]))
            for j, o in enumerate(ph):
                r.add(at[_fkey("p_flow", ln["id"], o, "ft")], mp[i][j])
                r.add(at[_fkey("q_flow", ln["id"], o, "ft")], mq[i][j])
                r.add(at[_fkey("w", ln["from_bus"], o)], -mp[i][j] * gf[j] + mq[i][j] * bf[j])
            rows.append(r.finish())
    return rows


def assemble_centralized(f: dict) -> dict:
    table = index_variables(f)
    at = {k: i for i, k in enumerate(table)}
    rows = build_power_balance(f, at) + build_load_model(f, at) + build_flow_equations(f, at)
    n = len(table)
    c, lo, hi = [0.0] * n, [-INF] * n, [INF] * n
    comp = {}
    for kind in ("generators", "buses", "lines"):
        for o in f[kind]:
            comp[(kind, o["id"])] = o
    for j, key in enumerate(table):
        parts = key.split(":")
        kind, owner, ph = parts[0], parts[1], int(parts[2])
        if kind in ("p_gen", "q_gen"):
            g = comp[("generators", owner)]
            pi = g["phases"].index(ph)
            if kind == "p_gen":
                c[j] = 1.0
                lo[j], hi[j] = _bound(g["p_lo"][pi], -INF), _bound(g["p_hi"][pi], INF)
            else:
                lo[j], hi[j] = _bound(g["q_lo"][pi], -INF), _bound(g["q_hi"][pi], INF)
        elif kind == "w":
            b = comp[("buses", owner)]
            pi = b["phases"].index(ph)
            lo[j], hi[j] = _bound(b["w_lo"][pi], -INF), _bound(b["w_hi"][pi], INF)
        elif kind in ("p_flow", "q_flow"):
            ln = comp[("lines", owner)]
            pi = ln["phases"].index(ph)
            pre = "p" if kind == "p_flow" else "q"
            lo[j], hi[j] = _bound(ln[pre + "_lo"][pi], -INF), _bound(ln[pre + "_hi"][pi], INF)
    return {"var_table": table, "rows": rows, "c": c, "x_lo": lo, "x_hi": hi}
