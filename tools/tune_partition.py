"""Feedback partition of the resident kernel (experiment): measure every CTA's
slack at the iteration's final barrier with the phase clock, shift cost shares
away from the CTAs without slack (the critical region), re-split, repeat.
usage: python tools/tune_partition.py [rounds] [beta] > log;  prints the best
DOPF_BLOCK_WEIGHTS string last."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08293_b200 import _native as N  # noqa: E402
from paper_2501_08293_b200 import dopf  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 6
beta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
f = dopf.synthetic_feeder("ieee8500", 8500)
_, _, model = dopf.load_model(f, workers=os.cpu_count() or 1)
model.precompute(os.cpu_count() or 1)
lib = N.cuda()
w = None
best = (1e9, None)
for r in range(rounds):
    if w is not None:
        os.environ["DOPF_BLOCK_WEIGHTS"] = ",".join(f"{x:.6f}" for x in w)
    s = dopf.CudaSolver(0)
    s.upload(model)
    G = s.info()["blocks"]
    if w is None:
        w = np.ones(G)
    ts = []
    for _ in range(6):
        res = s.solve(dopf.Settings(), outputs=False)
        ts.append(res.timings["solve"])
    per = 1e6 * min(ts[1:]) / res.iterations
    lib.dopf_cuda_set_profiling(s._h, 1)
    res = s.solve(dopf.Settings(), outputs=False)
    cyc = (N.i64 * (8 * G))()
    lib.dopf_cuda_phase_cycles(s._h, cyc, G)
    a = np.array(cyc[:], dtype=np.float64).reshape(G, 8) / res.iterations
    wait = a[:, 4]
    busy = a[:, [0, 1, 2, 3, 5]].sum(axis=1)
    print(f"round {r}: {per:.3f} us/iter ({1e6 / per:.0f} iter/s), iterations {res.iterations}, "
          f"wait min {wait.min():.0f} median {np.median(wait):.0f}, busy max {busy.max():.0f}", flush=True)
    if per < best[0]:
        best = (per, w.copy())
    w = w * (1.0 + beta * (wait - np.median(wait)) / np.median(busy))
    w = np.clip(w, 0.5, 1.5)
    w *= G / w.sum()
    del s
print("best", f"{best[0]:.3f} us/iter")
print(",".join(f"{x:.6f}" for x in best[1]))
