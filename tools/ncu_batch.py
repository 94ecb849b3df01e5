"""Batch solves of IEEE-123 load scenarios through the C ABI, for ncu
captures of the cluster-mode resident kernel (BASELINE configs[4] shape;
fewer scenarios than the bench so a full ncu replay stays short).

usage: python tools/ncu_batch.py [scenarios] [solves]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_08293_b200 import dopf, scenarios  # noqa: E402
from paper_2501_08293_b200.batch import BatchSolver  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 296
solves = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prep = dopf.CudaSolver(0)
models = scenarios.build_scenarios("ieee123", 123, range(count), gpu=prep)
bs = BatchSolver(0)
bs.upload(models)
for _ in range(solves):
    res = bs.solve(dopf.Settings(), outputs=False, trace=False)
its = [r.iterations for r in res]
print(f"{count} scenarios: iterations {min(its)}..{max(its)}, info {bs.info()}, bytes/iter {bs.bytes_per_iteration():.0f}")
