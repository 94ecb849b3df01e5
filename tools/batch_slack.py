"""Per-CTA-position slack of the batch kernel (phase clock over every
instance): is one of an instance's G CTAs systematically the slow one?
usage: python tools/batch_slack.py [scenarios] [shape]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08293_b200 import _native as N  # noqa: E402
from paper_2501_08293_b200 import dopf, scenarios  # noqa: E402
from paper_2501_08293_b200.batch import BatchSolver  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 296
shape = sys.argv[2] if len(sys.argv) > 2 else "ieee123"
models = scenarios.build_scenarios(shape, 123, range(count), gpu=dopf.CudaSolver(0))
bs = BatchSolver(0)
bs.upload(models)
bs.solve(dopf.Settings(), outputs=False, trace=False)
lib = N.cuda()
lib.dopf_cuda_set_profiling(bs._s._h, 1)
res = bs.solve(dopf.Settings(), outputs=False, trace=False)
G = bs.info()["blocks"]
nb = G * count
cyc = (N.i64 * (8 * nb))()
lib.dopf_cuda_phase_cycles(bs._s._h, cyc, nb)
its = np.array([r.iterations for r in res], dtype=np.float64)
a = np.array(cyc[:], dtype=np.float64).reshape(count, G, 8) / its[:, None, None]
names = ["target", "gemv", "dual", "eq+part", "wait", "x-upd"]
print(f"{shape} x {count}, G = {G}; per CTA position, median over instances (cycles/iter)")
for b in range(G):
    print(f"  CTA {b}: " + " ".join(f"{n} {np.median(a[:, b, q]):6.0f}" for q, n in enumerate(names)),
          f"busy {np.median(a[:, b, [0, 1, 2, 3, 5]].sum(axis=1)):6.0f}")
