"""Tuning-depth sweep for the resident split: rounds x beta -> best period
(one context each).  usage: python tools/tune_sweep.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08293_b200 import dopf  # noqa: E402

f = dopf.synthetic_feeder("ieee8500", 8500)
_, _, model = dopf.load_model(f, workers=os.cpu_count() or 1)
model.precompute(os.cpu_count() or 1)
for beta in ("0.5", "0.3", "0.8"):
    os.environ["DOPF_TUNE_BETA"] = beta
    for rounds in (8, 16, 24):
        s = dopf.CudaSolver(0)
        per = s.tune_partition(model, dopf.Settings(), rounds=rounds)
        ts = [s.solve(dopf.Settings(), outputs=False).timings["solve"] for _ in range(5)]
        print(f"beta {beta} rounds {rounds}: tuned {1e6 * per:.3f} us/iter, re-measured "
              f"{1e6 * min(ts) / 1237:.3f} us/iter ({1237 / min(ts):.0f} iter/s)", flush=True)
        del s
