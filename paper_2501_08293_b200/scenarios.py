"""Independent load scenarios of one feeder (BASELINE config 5) and their
sharding over ranks.

Each scenario is the base feeder with every load's (a, b) scaled by its own
seeded factor in [0.5, 1.5] (synth.cpp scale_loads); each is an independent
reference `solve` (admm.cpp:172-244) with its own iteration count. Sharding is
contiguous and balanced like the reference's `shard` (parallel.cpp:7-21):
scenario ranges per rank, no per-iteration collective (replicas).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
from typing import List, Tuple

from . import dopf


def shard(count: int, parts: int, index: int) -> Tuple[int, int]:
    """[begin, end) of part `index` of `count` items split into `parts`
    contiguous, balanced ranges (first count % parts ranges one longer) --
    the rule of reference parallel.cpp:7-21."""
    if parts < 1 or not 0 <= index < parts:
        raise ValueError("bad shard")
    base, extra = divmod(count, parts)
    begin = index * base + min(index, extra)
    return begin, begin + base + (1 if index < extra else 0)


def scenario_seed(seed: int, k: int) -> int:
    return seed * 1_000_003 + k


def build_scenarios(shape: str, seed: int, indices, workers: int = 0,
                    gpu: "dopf.CudaSolver" = None) -> List["dopf.DecomposedModel"]:
    """Decomposed + precomputed models of scenarios `indices`. Host C++ on
    `workers` threads; with `gpu` (a CudaSolver) the threads only assemble and
    partition, and the row reduction + operators of every scenario run in
    batched launches on the device (dopf.prepare_gpu, bitwise equal)."""
    base = dopf.synthetic_feeder(shape, seed)
    workers = workers or (os.cpu_count() or 1)

    def one(k):
        f = dopf.scale_loads(base, scenario_seed(seed, k))
        if gpu is not None:
            return dopf.partition(dopf.assemble_centralized(f), f)
        _, _, m = dopf.load_model(f)
        m.precompute()
        return m

    with cf.ThreadPoolExecutor(max_workers=workers) as ex:
        models = list(ex.map(one, list(indices)))
    if gpu is not None:
        dopf.prepare_gpu(models, gpu)
    return models
