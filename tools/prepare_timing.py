"""Setup time of the 4096-scenario batch (BASELINE configs[4]): host
decomposition + precompute on all cores vs host assemble/partition + the
batched GPU row reduction and operators (dopf.prepare_gpu).
Results are checked bitwise on a sample.  usage: python tools/prepare_timing.py [count]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08293_b200 import dopf, scenarios  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cores = os.cpu_count() or 1
solver = dopf.CudaSolver(0)
scenarios.build_scenarios("ieee123", 123, range(8), gpu=solver)  # warm-up (context, kernels)

t0 = time.perf_counter()
host = scenarios.build_scenarios("ieee123", 123, range(count))
t_host = time.perf_counter() - t0

import concurrent.futures as cf  # noqa: E402
base = dopf.synthetic_feeder("ieee123", 123)
t0 = time.perf_counter()
with cf.ThreadPoolExecutor(max_workers=cores) as ex:
    parts = list(ex.map(lambda k: (lambda f: dopf.partition(dopf.assemble_centralized(f), f))(
        dopf.scale_loads(base, scenarios.scenario_seed(123, k))), range(count)))
t_part = time.perf_counter() - t0
t0 = time.perf_counter()
secs = dopf.prepare_gpu(parts, solver)
t_gpu = time.perf_counter() - t0

for k in range(0, count, max(1, count // 16)):
    for name in ("A", "b", "P", "v"):
        assert np.array_equal(host[k].arr(name).view(np.uint64), parts[k].arr(name).view(np.uint64)), (k, name)
print(f"{count} IEEE-123 scenarios, {cores} host threads:")
print(f"  host decompose + precompute (threads):      {t_host:.3f} s")
print(f"  host assemble + partition only (threads):   {t_part:.3f} s")
print(f"  GPU row_reduce + operators (prepare_gpu):   {t_gpu:.3f} s "
      f"(pack/upload {secs['pack_s']:.3f}, kernels {secs['kernels_s']:.3f}, download/unpack {secs['unpack_s']:.3f})")
print(f"  GPU path total {t_part + t_gpu:.3f} s vs host {t_host:.3f} s; bitwise equal on 16 sampled scenarios")
