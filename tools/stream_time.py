"""Per-iteration time of the HBM-streaming path on the tiled feeder.

usage: python tools/stream_time.py [tiles] [iterations]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08293_b200 import dopf  # noqa: E402

tiles = int(sys.argv[1]) if len(sys.argv) > 1 else 64
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
t0 = time.time()
f = dopf.tiled_feeder("ieee8500", tiles, 850064)
_, _, model = dopf.load_model(f, workers=os.cpu_count() or 1)
model.precompute(os.cpu_count() or 1)
s = dopf.CudaSolver(0)
s.upload(model)
print(f"build+upload {time.time() - t0:.1f} s")
for _ in range(2):
    r = s.solve(dopf.Settings(max_iter=iters), outputs=False)
bpi = s.bytes_per_iteration()
us = 1e6 * r.timings["solve"] / r.iterations
print(f"tiled{tiles} DOPF_KLOCAL={os.environ.get('DOPF_KLOCAL', '0')}: {r.iterations} it, {us:.1f} us/iter, "
      f"{bpi / us / 1e3:.0f} GB/s algorithmic")
