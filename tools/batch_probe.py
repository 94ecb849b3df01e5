"""Batch of independent load scenarios on one GPU: timing + sampled parity.

usage: python tools/batch_probe.py [count] [shape] [seed]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle_py as O  # noqa: E402
from paper_2501_08293_b200 import dopf, scenarios  # noqa: E402
from paper_2501_08293_b200.batch import BatchSolver  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 256
shape = sys.argv[2] if len(sys.argv) > 2 else "ieee123"
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 123
t0 = time.time()
models = scenarios.build_scenarios(shape, seed, range(count))
t1 = time.time()
bs = BatchSolver(0)
bs.upload(models)
t2 = time.time()
st = dopf.Settings()
res = bs.solve(st, outputs=True, trace=False)
res = bs.solve(st, outputs=True, trace=False)
ksec = bs._s._lib.dopf_cuda_last_kernel_seconds(bs._s._h)
its = np.array([r.iterations for r in res])
print(f"{count} x {shape}: build {t1 - t0:.1f} s, upload {t2 - t1:.1f} s, info {bs.info()}")
print(f"kernel {ksec * 1e3:.2f} ms; iterations min {its.min()} median {int(np.median(its))} max {its.max()}; "
      f"sum {its.sum()} -> {its.sum() / ksec:.3e} scenario-iter/s; "
      f"batch-iterations/s {its.max() / ksec:.0f}; statuses {set(r.status for r in res)}")
bpi = bs.bytes_per_iteration() / count
print(f"algorithmic bytes: {bpi * its.sum() / ksec / 1e9:.1f} GB/s")
for k in sorted(set([0, count // 2, count - 1])):
    ref = O.solve(models[k], st)
    g = res[k]
    ok = (g.iterations == ref.iterations and np.array_equal(g.x, ref.x) and np.array_equal(g.z, ref.z)
          and np.array_equal(g.lam, ref.lam))
    print(f"scenario {k}: gpu {g.iterations} it, oracle {ref.iterations} it, bitwise {ok}")
