"""One solve of a synthetic feeder through the C ABI, for ncu captures.

usage: python tools/ncu_target.py [shape] [seed] [solves]

The model is built and uploaded first (host work, no kernels of ours), then
`solves` persistent-kernel launches run back to back; ncu's `-s` skips the
first ones (warm-up).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_08293_b200 import dopf  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "ieee8500"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 8500
solves = int(sys.argv[3]) if len(sys.argv) > 3 else 2
f = dopf.synthetic_feeder(shape, seed)
_, _, model = dopf.load_model(f, workers=os.cpu_count() or 1)
model.precompute(os.cpu_count() or 1)
s = dopf.CudaSolver(0)
s.upload(model)
for _ in range(solves):
    r = s.solve(dopf.Settings(), outputs=False)
print(f"{shape}: iterations={r.iterations} status={r.status} kernel={1e3 * r.timings['solve']:.3f} ms "
      f"info={s.info()} bytes/iter={s.bytes_per_iteration():.0f}")
