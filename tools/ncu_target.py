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
if os.environ.get("DOPF_TUNE") == "1":
    # the bench's slack-tuned split, exported for a profiler run of this tool
    # with DOPF_BLOCK_WEIGHTS=<the printed shares> (no tuning launches there)
    import ctypes as C
    s.tune_partition(model, dopf.Settings(), rounds=12)
    w = (C.c_double * 4096)()
    n = s._lib.dopf_cuda_block_weights(s._h, w, 4096)
    print("DOPF_BLOCK_WEIGHTS=" + ",".join(f"{w[i]:.9f}" for i in range(n)))
    sys.exit(0)
s.upload(model)
for _ in range(solves):
    r = s.solve(dopf.Settings(), outputs=False)
print(f"{shape}: iterations={r.iterations} status={r.status} kernel={1e3 * r.timings['solve']:.3f} ms "
      f"info={s.info()} bytes/iter={s.bytes_per_iteration():.0f}")
