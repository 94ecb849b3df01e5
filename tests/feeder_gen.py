"""Random radial feeders as feeder JSON, with the ranges of the reference's
test generator (proj/tests/test_util.hpp:77-172): 1-6 buses on a random phase
universe (phase 1 always present, the substation three-phase), each bus hung
off a random earlier bus through a line on the shared phases; diagonal
r in [0.01, 0.02], x in [0.02, 0.03], mutual r <= 0.002, x <= 0.004; line
shunts g <= 1e-3, b <= 2e-3; bus shunts <= 1e-2; w in [0.8, 0.9] x
[1.1, 1.2]; tap 1.0404 with probability 0.2; flow bounds +-2 or unbounded;
one generator at the root; loads on half of the non-root buses, on the
phases the feeding line serves (delta on three-phase lines w.p. 0.3),
a <= 0.2, b <= 0.1, alpha = beta in {0, 1, 2}.

`n_buses` lifts the size for scale tests (the reference draws 1-6)."""
from __future__ import annotations

import json

import numpy as np


def random_feeder(seed: int, n_buses: int = 0) -> str:
    rng = np.random.default_rng(seed)
    u = rng.random
    nb = n_buses or int(rng.integers(1, 7))
    width = len(str(max(nb - 1, 1)))
    bid = [f"bus{i:0{width}d}" for i in range(nb)]

    def phases():
        return [1] + [p for p in (2, 3) if u() < 0.6]

    buses, bph = [], []
    for i in range(nb):
        ph = [1, 2, 3] if i == 0 else phases()
        bph.append(ph)
        k = len(ph)
        buses.append({"id": bid[i], "phases": ph,
                      "w_lo": [0.8 + 0.1 * u() for _ in range(k)],
                      "w_hi": [1.1 + 0.1 * u() for _ in range(k)],
                      "g_sh": [0.01 * u() for _ in range(k)],
                      "b_sh": [0.01 * u() for _ in range(k)]})
    lines, lph = [], []
    for i in range(1, nb):
        parent = int(rng.integers(0, i))
        shared = [p for p in bph[i] if p in bph[parent]] or [bph[i][0]]
        lph.append(shared)
        k = len(shared)
        r = [[0.0] * k for _ in range(k)]
        x = [[0.0] * k for _ in range(k)]
        for a in range(k):
            for b in range(a, k):
                rv = 0.01 + 0.01 * u() if a == b else 0.002 * u()
                xv = 0.02 + 0.01 * u() if a == b else 0.004 * u()
                r[a][b] = r[b][a] = rv
                x[a][b] = x[b][a] = xv
        lines.append({"id": f"line{i:0{width}d}", "from_bus": bid[parent], "to_bus": bid[i],
                      "phases": shared, "r": r, "x": x,
                      "g_s_from": [0.001 * u() for _ in range(k)],
                      "b_s_from": [0.002 * u() for _ in range(k)],
                      "g_s_to": [0.001 * u() for _ in range(k)],
                      "b_s_to": [0.002 * u() for _ in range(k)],
                      "tau": [1.0404 if u() < 0.2 else 1.0 for _ in range(k)],
                      "p_lo": [None if u() < 0.5 else -2.0 for _ in range(k)],
                      "p_hi": [None if u() < 0.5 else 2.0 for _ in range(k)],
                      "q_lo": [-2.0] * k, "q_hi": [2.0] * k})
    gens = [{"id": "gen0", "bus": bid[0], "phases": [1, 2, 3], "p_lo": [0.0] * 3, "p_hi": [5.0] * 3,
             "q_lo": [-5.0] * 3, "q_hi": [5.0] * 3}]
    loads = []
    for i in range(1, nb):
        if u() < 0.5:
            continue
        served = lph[i - 1]
        delta = len(served) == 3 and u() < 0.3
        k = len(served)
        e = [float(rng.integers(0, 3)) for _ in range(k)]
        loads.append({"id": f"load{i:0{width}d}", "bus": bid[i], "connection": "delta" if delta else "wye",
                      "phases": served, "a": [0.2 * u() for _ in range(k)],
                      "b": [0.1 * u() for _ in range(k)], "alpha": e, "beta": list(e)})
    return json.dumps({"base": 1.0 + 99.0 * u(), "buses": buses, "generators": gens,
                       "lines": lines, "loads": loads})
