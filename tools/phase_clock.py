"""Per-phase SM-cycle breakdown of the persistent kernel, every CTA.

usage: python tools/phase_clock.py [shape] [seed]

Compute-warp phases are timed by warp 1 lane 0 of each CTA (they include the
barrier waits that end each phase); service phases by warp 0 lane 0.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_08293_b200 import _native as N  # noqa: E402
from paper_2501_08293_b200 import dopf  # noqa: E402

PHASES = ["target", "gemv", "dual+publish", "eq+partials", "exch-wait", "x-update",
          "svc:nbr-wait", "svc:all+comb"]

shape = sys.argv[1] if len(sys.argv) > 1 else "ieee8500"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 8500
f = dopf.synthetic_feeder(shape, seed)
_, _, model = dopf.load_model(f, workers=8)
model.precompute(8)
s = dopf.CudaSolver(0)
s.upload(model)
lib = N.cuda()
s.solve(dopf.Settings())
lib.dopf_cuda_set_profiling(s._h, 1)
r = s.solve(dopf.Settings())
G = s.info()["blocks"] * s.info()["instances"]
cyc = (N.i64 * (8 * G))()
lib.dopf_cuda_phase_cycles(s._h, cyc, G)
a = np.array(cyc[:], dtype=np.float64).reshape(G, 8) / r.iterations
print(f"{shape}: {r.iterations} iterations, kernel {1e3 * r.timings['solve']:.3f} ms, "
      f"{1e6 * r.timings['solve'] / r.iterations:.2f} us/iter, info {s.info()}")
print(f"  {'phase':14s} {'CTA0':>8s} {'min':>8s} {'median':>8s} {'max':>8s} {'argmax':>6s}  (cycles/iter)")
for q, name in enumerate(PHASES):
    col = a[:, q]
    print(f"  {name:14s} {col[0]:8.0f} {col.min():8.0f} {np.median(col):8.0f} {col.max():8.0f} "
          f"{int(col.argmax()):6d}")
busy = a[:, [0, 1, 2, 3, 5]].sum(axis=1)
if os.environ.get("PHASE_DUMP"):  # per-CTA busy cycles + layout statistics for a cost-model fit
    st = (N.i64 * (12 * G))()
    lib.dopf_cuda_block_stats(s._h, st, G)
    np.savez(os.environ["PHASE_DUMP"], phases=a, stats=np.array(st[:], dtype=np.int64).reshape(G, 12))
print(f"  compute (no exch-wait): min {busy.min():.0f} median {np.median(busy):.0f} "
      f"max {busy.max():.0f} (CTA {int(busy.argmax())})")

# cross-CTA timeline (globaltimer, ns) for iterations 100..163
T = 64
buf = (N.u64 * (G * T * 3))()
if lib.dopf_cuda_timeline(s._h, buf, G * T * 3) == 0:
    tl = np.array(buf[:], dtype=np.float64).reshape(G, T, 3)
    ok = tl[:, :, 0] > 0
    if ok.any():
        t0 = tl[:, :, 0][ok].min()
        pub = tl[:, :, 0] - t0
        per = np.diff(pub, axis=1)
        print(f"timeline: iteration period median {np.median(per):.0f} ns; "
              f"publish skew across CTAs per iteration: median {np.median(pub.max(0) - pub.min(0)):.0f} ns, "
              f"max {np.max(pub.max(0) - pub.min(0)):.0f} ns")
        wait = tl[:, :, 2] - tl[:, :, 1]
        gap = tl[:, :, 1] - tl[:, :, 0]
        print(f"  publish -> boundary start: median {np.median(gap):.0f} ns; boundary update: median "
              f"{np.median(wait):.0f} ns, p90 {np.percentile(wait, 90):.0f}, max {wait.max():.0f}")
        late = np.argsort(-np.median(pub - pub.min(0), axis=1))[:5]
        print("  latest publishers (CTA: median lag ns):",
              ", ".join(f"{g}: {np.median(pub[g] - pub.min(0)):.0f}" for g in late))
        print("  globaltimer distinct deltas (resolution probe):", np.unique(np.diff(np.sort(tl[0, :, 0])))[:5])
