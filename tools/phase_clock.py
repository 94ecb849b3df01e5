"""Per-phase SM-cycle breakdown of the persistent kernel (CTA 0, thread 0).

usage: python tools/phase_clock.py [shape] [seed]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_08293_b200 import _native as N  # noqa: E402
from paper_2501_08293_b200 import dopf  # noqa: E402

PHASES = ["top-wait", "target", "gemv", "eq+dual", "reduce", "exchange", "x-update", "combine"]

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
cyc = (N.i64 * 8)()
lib.dopf_cuda_phase_cycles(s._h, cyc)
tot = sum(cyc)
print(f"{shape}: {r.iterations} iterations, kernel {1e3 * r.timings['solve']:.3f} ms, "
      f"{1e6 * r.timings['solve'] / r.iterations:.2f} us/iter, info {s.info()}")
for name, c in zip(PHASES, cyc):
    print(f"  {name:10s} {c / r.iterations:10.0f} cycles/iter  {100.0 * c / max(tot, 1):5.1f}%")
