"""Same-structure re-upload cost of the IEEE-8500 model (the e2e arm's per-step
upload): the C-ABI call vs a raw pinned copy of the same bytes.
usage: python tools/upload_timing.py"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_08293_b200 import _native as N  # noqa: E402
from paper_2501_08293_b200 import dopf  # noqa: E402

f = dopf.synthetic_feeder("ieee8500", 8500)
_, _, model = dopf.load_model(f, workers=os.cpu_count() or 1)
model.precompute(os.cpu_count() or 1)
s = dopf.CudaSolver(0)
s.tune_partition(model, dopf.Settings(), rounds=4)
s.pin(model)
v = model.view()
lib = N.cuda()
for _ in range(3):
    lib.dopf_cuda_upload(s._h, C.byref(v))
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    lib.dopf_cuda_upload(s._h, C.byref(v))
    ts.append(time.perf_counter() - t0)
st = model.stats()
nbytes = 8 * (st["sum_n2"] + st["sum_mn"] + st["sum_m"] + 2 * st["N_z"] + 4 * st["n"])
h = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(h, device="cuda")
torch.cuda.synchronize()
tc = []
for _ in range(20):
    t0 = time.perf_counter()
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    tc.append(time.perf_counter() - t0)
print(f"upload (same structure, pinned): median {1e3 * sorted(ts)[10]:.3f} ms for {nbytes / 1e6:.1f} MB; "
      f"one raw pinned copy of the same bytes: {1e3 * sorted(tc)[10]:.3f} ms "
      f"({nbytes / sorted(tc)[10] / 1e9:.1f} GB/s)")
