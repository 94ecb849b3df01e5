"""Fit the resident kernel's per-CTA compute cycles (phase clock) to layout
statistics (dopf_cuda_block_stats), to calibrate the block-splitting cost.
usage: python tools/fit_block_cost.py dump.npz"""
import sys

import numpy as np

d = np.load(sys.argv[1])
a, st = d["phases"], d["stats"].astype(np.float64)
names = ["rows", "cols", "cols_int", "arows", "p_len", "a_len", "copy_len", "nbr_cnt", "remote", "exported",
         "chain", "sum_n"]
busy = a[:, [0, 1, 2, 3, 5]].sum(axis=1)
print(f"busy cycles/iter: min {busy.min():.0f} median {np.median(busy):.0f} max {busy.max():.0f}")
for q, nm in enumerate(names):
    c = np.corrcoef(st[:, q], busy)[0, 1]
    print(f"  {nm:9s} mean {st[:, q].mean():10.1f} sd {st[:, q].std():9.1f} corr(busy) {c:+.2f}")
for phase, q in (("gemv", 1), ("dual", 2), ("eq+partials", 3), ("x-update", 5)):
    best = max(range(len(names)), key=lambda k: abs(np.corrcoef(st[:, k], a[:, q])[0, 1]))
    print(f"  phase {phase:11s} median {np.median(a[:, q]):6.0f} sd {a[:, q].std():5.0f}  best predictor {names[best]} "
          f"({np.corrcoef(st[:, best], a[:, q])[0, 1]:+.2f})")
X = np.column_stack([np.ones(len(busy)), st[:, [0, 4, 5, 1, 8, 10]]])
coef, *_ = np.linalg.lstsq(X, busy, rcond=None)
pred = X @ coef
print("fit busy ~ 1 + rows + p_len + a_len + cols + remote + chain:", np.round(coef, 3))
print(f"  residual sd {np.std(busy - pred):.0f} cycles (busy sd {busy.std():.0f})")
