"""A few streaming-path iterations of the tiled feeder, for ncu captures.

usage: python tools/ncu_tiled.py [tiles] [iterations]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_08293_b200 import dopf  # noqa: E402

tiles = int(sys.argv[1]) if len(sys.argv) > 1 else 16
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
f = dopf.tiled_feeder("ieee8500", tiles, 850064)
_, _, model = dopf.load_model(f, workers=os.cpu_count() or 1)
model.precompute(os.cpu_count() or 1)
s = dopf.CudaSolver(0)
s.upload(model)
r = s.solve(dopf.Settings(max_iter=iters), outputs=False)
print(f"tiled{tiles}: {r.iterations} iterations, {1e3 * r.timings['solve']:.2f} ms, info {s.info()}, "
      f"bytes/iter {s.bytes_per_iteration():.0f}")
