"""Benchmark of the B200 ADMM hot path (BASELINE.json metric: ADMM iters/sec &
time-to-converge, IEEE 8500-bus; HBM GB/s vs peak).

A "step" is one complete solve to convergence (reference dopf::solve,
admm.cpp:172-244) of the configured workload (rho = 100, eps_rel = 1e-3,
max_iter = 50000, the paper's settings):

  --config ieee8500  (default) the synthetic IEEE-8500-shape feeder, one
                     instance per GPU (BASELINE configs[2], the metric's case)
  --config ieee123 / ieee13   single instances of the smaller shapes
  --config batch123  --scenarios K independent load scenarios of the
                     IEEE-123 shape (configs[4]), sharded over ranks
  --config tiled     --tiles T copies of the IEEE-8500 shape tied to one root
                     (configs[3], T = 64: ~0.76M nodes, 10.8M local variables),
                     solved on the HBM-streaming path

Line keys:
  value     ADMM iterations / second on the device: iterations of the K timed
            solves (summed over scenarios for a batch) / their kernel time
            (CUDA events on the launching stream); inputs resident in HBM;
            L2 flushed (256 MiB write) between solves. N > 1: whole job, time =
            max over ranks.
  e2e       the same metric through the reference-facing C ABI with HOST
            buffers: dopf_cuda_upload(_batch) (host model -> HBM layout) +
            dopf_cuda_solve(_batch) (x / z / lambda / trace copied back into
            host buffers) per step.
  roofline  algorithmic bytes (B_iter per iteration x
            iterations of one launch) / kernel time, against
            MEASURED_PEAKS.json hbm_gbs; traffic = ncu DRAM bytes per launch.
  cpu_baseline  the CPU oracle (C++ restatement of the reference loop, all
            host threads) on a bounded sample of the same workload.

--impl reference times the reference's CPU path (the oracle port -- the C++
reference cannot be built here) on the same config and
metric. Multi-GPU (torchrun, N > 1): ieee8500 runs one independent load
scenario per rank; batch123 shards the scenarios (no per-iteration
collective); tiled splits ONE instance by subtree over the ranks with an NCCL
all-gather of the boundary copies every iteration ("strong").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SINGLE = {"ieee8500": 8500, "ieee123": 123, "ieee13": 13}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="ieee8500", choices=sorted(SINGLE) + ["batch123", "tiled"])
    ap.add_argument("--tiles", type=int, default=64, help="tiled: IEEE-8500 copies")
    ap.add_argument("--shape", default=None, help="alias of --config for single instances")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--scenarios", type=int, default=4096, help="batch123: total scenarios")
    ap.add_argument("--cpu-sample-iters", type=int, default=0,
                    help="iterations per CPU sample (0: auto, ~10-30 s of CPU work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.shape:
        args.config = args.shape
    if args.seed is None:
        args.seed = SINGLE.get(args.config, 850064 if args.config == "tiled" else 123)
    return args


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("DOPF_SHARE_GPU") == "1":  # test knob: every rank on device 0 (gloo)
        local = 0
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ workloads


def build_models(args, rank, world, workers):
    """The rank's models: [one instance] or [its shard of the scenarios]."""
    from paper_2501_08293_b200 import dopf, scenarios
    if args.config == "batch123":
        b, e = scenarios.shard(args.scenarios, world, rank)
        return scenarios.build_scenarios("ieee123", args.seed, range(b, e), workers)
    if args.config == "tiled":
        f = dopf.tiled_feeder("ieee8500", args.tiles, args.seed)
    else:
        f = dopf.synthetic_feeder(args.config, args.seed)
    if rank > 0:  # weak scaling: rank r solves load scenario r of the same feeder
        f = dopf.scale_loads(f, scenarios.scenario_seed(args.seed, rank))
    _, _, model = dopf.load_model(f, workers=workers)
    model.precompute(workers)
    return [model]


def metric_name(args):
    if args.config == "batch123":
        return "admm_iterations_per_second_batch4096_ieee123"
    if args.config == "tiled":
        return f"admm_iterations_per_second_ieee8500_tiled{args.tiles}"
    return "admm_iterations_per_second_" + args.config


def config_of(args, world):
    if args.config == "batch123":
        w = (f"{args.scenarios} independent load scenarios of the synthetic ieee123 feeder "
             f"(seed {args.seed}, loads scaled U[0.5,1.5]), each solved to convergence "
             "(rho=100, eps_rel=1e-3, max_iter=50000); value = scenario-iterations/s")
        par = f"scenario-sharded over {world} rank(s)" if world > 1 else "single-gpu"
    elif args.config == "tiled":
        w = (f"{args.tiles} synthetic ieee8500 feeders (seed {args.seed}) tied by 3-phase tie lines "
             "to one root bus, one instance, solve to convergence (rho=100, eps_rel=1e-3, "
             "max_iter=50000), HBM-streaming CUDA-graph path")
        par = "independent scenario per rank" if world > 1 else "single-gpu"
    else:
        w = (f"{args.config} synthetic feeder (seed {args.seed}), single instance per GPU, "
             "solve to convergence (rho=100, eps_rel=1e-3, max_iter=50000)")
        par = "independent scenario per rank" if world > 1 else "single-gpu"
    return {"workload": w, "parallelism": par, "l2": "flushed (256 MiB write) between timed solves"}


def cpu_sample(models, settings_kw, sample_iters, workers):
    """Oracle (restated reference CPU path): iterations/s on a bounded sample.
    A batch is sampled scenario-parallel (one thread per scenario)."""
    import concurrent.futures as cf

    from oracle import oracle_py as O
    from paper_2501_08293_b200 import dopf
    if len(models) == 1:
        st = dopf.Settings(**{**settings_kw, "max_iter": sample_iters, "workers": workers})
        t0 = time.perf_counter()
        r = O.solve(models[0], st)
        dt = time.perf_counter() - t0
        return r.iterations / dt, r.iterations, dt, 1
    sample = models[:workers]
    st = dopf.Settings(**{**settings_kw, "max_iter": sample_iters, "workers": 1})
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=len(sample)) as ex:
        its = sum(r.iterations for r in ex.map(lambda m: O.solve(m, st), sample))
    dt = time.perf_counter() - t0
    return its / dt, its, dt, len(sample)


def auto_cpu_iters(models, workers, settings_kw, target_s=12.0):
    it_s, its, dt, n = cpu_sample(models, settings_kw, 20, workers)
    per_scen = it_s / max(1, n)
    return max(20, min(50000, int(per_scen * target_s)))


def cpu_model() -> str:
    """Host CPU model name (/proc/cpuinfo, as lscpu prints it)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


NCU_TARGETS = {"ieee8500": ("ieee8500", 8500), "ieee123": ("ieee123", 123), "ieee13": ("ieee13", 13)}


def ncu_traffic(config: str):
    """DRAM bytes (read + write) of one launch of the resident kernel,
    measured now: ncu on tools/ncu_target.py (the same model, one warm-up
    launch skipped). None when ncu is missing or the capture fails."""
    if config not in NCU_TARGETS or os.environ.get("DOPF_BENCH_NO_NCU"):
        return None, "skipped"
    ncu = "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    shape, seed = NCU_TARGETS[config]
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none",
           "-k", "regex:admm_persistent", "-s", "1", "-c", "1", "--csv", "--print-units", "base",
           sys.executable, os.path.join(ROOT, "tools", "ncu_target.py"), shape, str(seed), "2"]
    try:
        out = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                             timeout=240).stdout
    except Exception as e:  # noqa: BLE001
        return None, f"ncu failed: {type(e).__name__}"
    import csv
    tot, seen = 0.0, 0
    for row in csv.reader(line for line in out.splitlines() if "dram__bytes_" in line):
        if len(row) >= 2 and row[-3 if len(row) >= 3 else 0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            try:
                tot += float(row[-1].replace(",", ""))
                seen += 1
            except ValueError:
                pass
    return (tot if seen == 2 else None), ("ncu live capture (dram__bytes_read.sum + dram__bytes_write.sum, "
                                          "one launch)" if seen == 2 else "ncu output unparsed")


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def run_reference(args, rank, world):
    """The reference's CPU path (oracle port) on this config: rank 0 only."""
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    settings_kw = dict(rho=100.0, eps_rel=1e-3)
    if args.config == "batch123":
        from paper_2501_08293_b200 import scenarios
        models = scenarios.build_scenarios("ieee123", args.seed, range(workers), workers)
    else:
        models = build_models(args, 0, 1, workers)
    iters = args.cpu_sample_iters or auto_cpu_iters(models, workers, settings_kw, target_s=8.0)
    for _ in range(args.warmup):
        cpu_sample(models, settings_kw, max(5, iters // 10), workers)
    tot_it, tot_t, n = 0, 0.0, 1
    for _ in range(args.steps):
        _, it, dt, n = cpu_sample(models, settings_kw, iters, workers)
        tot_it += it
        tot_t += dt
    value = tot_it / tot_t
    per_step = tot_it / max(1, args.steps)
    if n > 1:
        what = (f"{per_step:.0f} ADMM iterations over {n} scenarios (one thread per scenario, each "
                f"capped at {iters} iterations)")
    else:
        what = (f"{per_step:.0f} ADMM iterations of the {args.config} solve (WorkerPool of {workers} "
                f"threads; cap {iters}" + (", the solve stops at convergence first)" if per_step < iters else ")"))
    line = {
        "impl": "reference",
        "metric": metric_name(args),
        "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of(args, world),
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": workers, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": what + " per step; C++ oracle restating admm.cpp:172-244"},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def upload_bytes(models, batch: bool = False) -> int:
    """Bytes the per-step upload copies host -> device. A single model after
    its first upload takes the same-structure path: the raw value arrays only
    (P, A, b, v, z0, c, 1/copies, lo, hi), scattered on the device. A batch
    upload copies its device layout (estimated from the model sizes)."""
    if not batch:
        tot = 0
        for model in models:
            st = model.stats()
            tot += 8 * (st["sum_n2"] + st["sum_mn"] + st["sum_m"] + 2 * st["N_z"] + 4 * st["n"])
        return int(tot)
    tot = 0
    for model in models:
        st = model.stats()
        Nz = st["N_z"]
        ops = 8 * (st["sum_n2"] + st["sum_mn"])
        rows = Nz * (16 + 8 + 8)            # RowMeta + v + z0
        cols = Nz * (16 + 32) + 4 * Nz      # column metadata (upper bound) + copies
        arow = st["sum_m"] * (16 + 8)
        tot += int(ops + rows + cols + arow + 80 * 148)
    return tot


def run_partitioned(args, rank, world, local):
    """Tiled feeder split by subtree over `world` GPUs (strong scaling): one
    instance, one gather of the packed boundary records per iteration. On
    GPUs (NCCL) the library drives it itself: dopf_cuda_comm_init +
    dopf_cuda_solve_part, the whole loop -- kernels and ncclAllGather -- one
    CUDA graph per solve. Ranks sharing one GPU (tests, gloo) step the same
    kernels through torch.distributed (partition.PartitionedSolver)."""
    import numpy as np
    import torch
    import torch.distributed as td

    from paper_2501_08293_b200 import dopf
    from paper_2501_08293_b200.partition import NcclPartitionedSolver, PartitionedSolver
    torch.cuda.set_device(local)
    workers = max(1, (os.cpu_count() or 1) // max(1, world))
    f = dopf.tiled_feeder("ieee8500", args.tiles, args.seed)
    _, _, model = dopf.load_model(f, workers=workers)
    model.precompute(workers)
    capi = td.get_backend() == "nccl" and os.environ.get("DOPF_PART_IMPL", "capi") == "capi"
    ps = NcclPartitionedSolver.from_torch_distributed(local) if capi else PartitionedSolver(local)
    if os.environ.get("DOPF_BENCH_PAGEABLE") != "1":
        ps.solver.pin(model)  # e2e inputs from pinned host memory (setup)
    ps.upload(model)
    settings = dopf.Settings(rho=100.0, eps_rel=1e-3, max_iter=50000)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")
    lib = ps.solver._lib

    def timed_solve(trace=False):
        if capi:  # CUDA events around the graph on the solver's stream (inside the library)
            r = ps.solve(settings, trace=trace)
            return r, float(lib.dopf_cuda_last_kernel_seconds(ps.solver._h))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ps.stream)
        r = ps.solve(settings, trace=trace)
        e1.record(ps.stream)
        e1.synchronize()
        return r, e0.elapsed_time(e1) * 1e-3

    for _ in range(max(3, args.warmup)):
        timed_solve()
    times, its = [], []
    k0 = ps.solver.kernels_executed()
    with ClockSampler(local) as clocks:
        td.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            r, dt = timed_solve()
            times.append(dt)
            its.append(r.iterations)
        td.barrier()
        torch.cuda.synchronize()
    kernels = ps.solver.kernels_executed() - k0
    t = torch.tensor([sum(times), ps.bytes_per_iteration()], dtype=torch.float64, device=f"cuda:{local}")
    allt = [torch.zeros_like(t) for _ in range(world)]
    td.all_gather(allt, t)
    max_t = max(float(a[0]) for a in allt)
    bytes_job = sum(float(a[1]) for a in allt)
    value = sum(its) / max_t
    # e2e per rank: upload of the whole model (host layout + H2D of its share)
    # + solve + its share of x / z / lambda and the trace back in host memory
    e2e_t, e2e_it = 0.0, 0
    for step in range(args.steps + 1):
        td.barrier()
        t0 = time.perf_counter()
        ps.upload(model)
        r = ps.solve(settings, trace=True)
        dt = time.perf_counter() - t0
        if step > 0:
            e2e_t += dt
            e2e_it += r.iterations
    tt = torch.tensor([e2e_t], dtype=torch.float64, device=f"cuda:{local}")
    td.all_reduce(tt, op=td.ReduceOp.MAX)
    peak, peak_kind = read_peaks()
    achieved = bytes_job * (sum(its) / args.steps) / (max_t / args.steps) / 1e9
    mode = ps.graph_mode() if capi else "torch.distributed steps"
    if rank == 0:
        st = model.stats()
        line = {
            "metric": metric_name(args), "value": value, "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": 1e3 * max_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {**config_of(args, world), "parallelism": f"subtree-partitioned over {world} GPUs "
                       "(one NCCL all-gather of the packed [boundary u | residual partials] records per "
                       f"iteration; loop: {mode})"},
            "time_to_converge_ms": 1e3 * max_t / args.steps, "iterations_to_converge": int(its[-1]),
            "status": "converged" if r.status == 0 else "iteration_limit", "objective": r.objective,
            "e2e": {"value": e2e_it / float(tt[0]), "unit": "iter/s",
                    "h2d_bytes_per_step": int(8 * (st["sum_n2"] + st["sum_mn"]) + 40 * st["N_z"]),
                    "d2h_bytes_per_step": int(8 * (st["n"] + 2 * st["N_z"])),
                    "time_to_converge_ms": 1e3 * float(tt[0]) / args.steps,
                    "note": "per rank: upload + solve + its share of the results to host memory; "
                            "max over ranks"},
            "gpu_launches": int(kernels),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                         "frac": achieved / (peak * world), "traffic": None, "peak_kind": peak_kind,
                         "bytes_per_iteration": bytes_job,
                         "note": "whole job: algorithmic bytes of all ranks / max rank time vs world x HBM peak"},
            "kernel": {"name": "k_global+k_staged(+k_local)+k_pack+ncclAllGather+k_decide per iteration",
                       "ranks": world, "driver": "C ABI dopf_cuda_solve_part" if capi else "python"},
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    rank, world, local = dist_env()
    import torch
    # DOPF_BENCH_PARTITIONED=1: the partitioned tiled path even at one rank
    # (under torchrun; exercises the NCCL loop on a one-GPU box)
    part_one = args.config == "tiled" and os.environ.get("DOPF_BENCH_PARTITIONED") == "1"
    if world > 1 or part_one:
        import torch.distributed as td
        shared = os.environ.get("DOPF_SHARE_GPU") == "1"  # NCCL refuses two ranks on one GPU
        backend = os.environ.get("DOPF_DIST_BACKEND") or (
            "nccl" if torch.cuda.is_available() and not shared else "gloo")
        td.init_process_group(backend=backend)
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            import torch.distributed as td
            td.destroy_process_group()
        return
    if args.config == "tiled" and (world > 1 or part_one):
        run_partitioned(args, rank, world, local)
        import torch.distributed as td
        td.destroy_process_group()
        return

    import ctypes as C

    import numpy as np

    from paper_2501_08293_b200 import _native as N
    from paper_2501_08293_b200 import dopf

    device = local
    torch.cuda.set_device(device)
    workers = max(1, (os.cpu_count() or 1) // max(1, world))
    models = build_models(args, rank, world, workers)
    batch = args.config == "batch123"
    settings = dopf.Settings(rho=100.0, eps_rel=1e-3, max_iter=50000)
    st = settings.to_c()
    lib = N.cuda()
    solver = dopf.CudaSolver(device)
    # the e2e arm copies each step's inputs from pinned host memory: page-lock
    # the models' value arrays once (setup, outside every timed region)
    pinned = os.environ.get("DOPF_BENCH_PAGEABLE") != "1"
    if pinned:
        for m in models:
            solver.pin(m)
    views = (N.ModelView_t * len(models))(*[m.view() for m in models])

    def upload():
        if batch:
            return lib.dopf_cuda_upload_batch(solver._h, views, len(models))
        return lib.dopf_cuda_upload(solver._h, C.byref(views[0]))

    rc = upload()
    if rc != 0:
        raise RuntimeError(lib.dopf_cuda_last_error(solver._h).decode())
    # setup (untimed): slack-tuned split of the resident single-instance
    # kernel, kept by the context for every later upload of this structure
    tuned_period = None
    # (DOPF_TUNE_BATCH=1 also tunes a batch's CTA split on a sample: measured
    # no faster for the tight 4-CTA IEEE-123 instances, so off by default)
    if os.environ.get("DOPF_NO_TUNE") != "1" and (not batch or os.environ.get("DOPF_TUNE_BATCH") == "1"):
        if batch:  # on a sample of two scenarios per CTA group, then the whole batch again
            sample = (N.ModelView_t * min(len(models), 74))(*[views[i] for i in range(min(len(models), 74))])
            per = C.c_double(0.0)
            if lib.dopf_cuda_tune_partition_batch(solver._h, sample, len(sample), C.byref(st), 6, C.byref(per)) != 0:
                raise RuntimeError(lib.dopf_cuda_last_error(solver._h).decode())
            tuned_period = per.value or None
            if upload() != 0:
                raise RuntimeError(lib.dopf_cuda_last_error(solver._h).decode())
        else:
            tuned_period = solver.tune_partition(models[0], settings, rounds=12) or None
    info = solver.info()
    b_iter = solver.bytes_per_iteration() / len(models)   # one instance
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{device}")  # 256 MiB
    K = len(models)

    def device_solve():
        rs = (N.ResultView_t * K)()
        if batch:
            rc = lib.dopf_cuda_solve_batch(solver._h, C.byref(st), rs, K)  # scalars only (null vectors)
        else:
            rc = lib.dopf_cuda_solve_device(solver._h, C.byref(st), rs)
        if rc != 0:
            raise RuntimeError(lib.dopf_cuda_last_error(solver._h).decode())
        its = [rs[i].iterations for i in range(K)]
        return its, [rs[i].status for i in range(K)], lib.dopf_cuda_last_kernel_seconds(solver._h), \
            rs[0].objective

    for _ in range(max(3, args.warmup)):
        device_solve()

    def barrier():
        if world > 1:
            import torch.distributed as td
            td.barrier()
        torch.cuda.synchronize()

    launches0 = solver.kernel_launches()
    kernels0 = solver.kernels_executed()
    per_step = []
    with ClockSampler(device) as clocks:
        barrier()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            per_step.append(device_solve())
        barrier()
    launches = solver.kernel_launches() - launches0
    kernels = solver.kernels_executed() - kernels0
    iters = [sum(p[0]) for p in per_step]
    ktime = [p[2] for p in per_step]
    tot_it, tot_t = sum(iters), sum(ktime)
    max_t = tot_t
    if world > 1:
        import torch.distributed as td
        t = torch.tensor([tot_t, float(tot_it)], dtype=torch.float64, device=f"cuda:{device}")
        all_t = [torch.zeros_like(t) for _ in range(world)]
        td.all_gather(all_t, t)
        max_t = max(float(a[0]) for a in all_t)
        tot_it = sum(float(a[1]) for a in all_t)
    value = tot_it / max_t

    # end-to-end through the C ABI with host buffers (upload + solve + copies)
    outs = []
    for m in models:
        v = m.view()
        outs.append((np.zeros(v.n), np.zeros(v.N_z), np.zeros(v.N_z), np.zeros((settings.max_iter, 6))))
        if pinned:  # result buffers page-locked too (setup)
            for a in outs[-1]:
                solver.pin_array(a)
    e2e_t, e2e_it = 0.0, 0
    for step in range(args.steps + 1):
        rs = (N.ResultView_t * K)()
        for i, (x, z, lam, tr) in enumerate(outs):
            rs[i].x = x.ctypes.data_as(C.POINTER(C.c_double))
            rs[i].z = z.ctypes.data_as(C.POINTER(C.c_double))
            rs[i].lambda_ = lam.ctypes.data_as(C.POINTER(C.c_double))
            rs[i].trace = tr.ctypes.data_as(C.POINTER(C.c_double))
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = upload()
        t_up = time.perf_counter() - t0
        if rc == 0:
            rc = (lib.dopf_cuda_solve_batch(solver._h, C.byref(st), rs, K) if batch
                  else lib.dopf_cuda_solve(solver._h, C.byref(st), rs))
        dt = time.perf_counter() - t0
        if rank == 0 and step == args.steps:
            print(f"e2e step: upload {1e3 * t_up:.1f} ms, solve+copies {1e3 * (dt - t_up):.1f} ms "
                  f"(kernel {1e3 * lib.dopf_cuda_last_kernel_seconds(solver._h):.1f} ms)",
                  file=sys.stderr, flush=True)
        if rc != 0:
            raise RuntimeError(lib.dopf_cuda_last_error(solver._h).decode())
        if step > 0:  # first pass warms the host allocator
            e2e_t += dt
            e2e_it += sum(rs[i].iterations for i in range(K))
    h2d = upload_bytes(models, batch)
    d2h = sum(8 * (m.view().n + 2 * m.view().N_z) + 32 for m in models) + 48 * int(np.mean(iters))
    e2e_value = e2e_it / e2e_t
    if world > 1:
        import torch.distributed as td
        t = torch.tensor([e2e_t, float(e2e_it)], dtype=torch.float64, device=f"cuda:{device}")
        all_t = [torch.zeros_like(t) for _ in range(world)]
        td.all_gather(all_t, t)
        e2e_value = sum(float(a[1]) for a in all_t) / max(float(a[0]) for a in all_t)

    peak, peak_kind = read_peaks()
    kernel_avg = tot_t / args.steps
    achieved = b_iter * (sum(iters) / args.steps) / kernel_avg / 1e9
    traffic, traffic_src = (None, "not measured (N > 1)")
    if rank == 0 and world == 1:
        traffic, traffic_src = ncu_traffic(args.config)
    if traffic is None:
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            try:
                with open(tp) as fh:
                    traffic = json.load(fh).get(args.config)
                if traffic is not None:
                    traffic_src += "; committed profiles/ncu_traffic.json (ncu --set full of the same command)"
            except Exception:
                traffic = None
    last_its, last_status = per_step[-1][0], per_step[-1][1]

    if rank == 0:
        line = {
            "metric": metric_name(args),
            "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": 1e3 * max_t / args.steps,
            "higher_is_better": True, "scaling": "strong" if (batch and world > 1) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_of(args, world),
            "time_to_converge_ms": 1e3 * kernel_avg,
            "iterations_to_converge": int(round(np.median(last_its))) if batch else int(last_its[0]),
            "status": "converged" if all(s == 0 for s in last_status) else "iteration_limit",
            "objective": per_step[-1][3],
            "e2e": {"value": e2e_value, "unit": "iter/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "time_to_converge_ms": 1e3 * e2e_t / args.steps,
                    "host_memory": "pinned (cudaHostRegister of the model value arrays and result buffers)"
                    if pinned else "pageable"},
            "gpu_launches": int(kernels),
            "graph_or_kernel_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_kind": peak_kind, "bytes_per_iteration": b_iter,
                         "traffic_per": "launch" if info["sync"] != "stream-graph" else "iteration",
                         "note": "algorithmic bytes (DESIGN.md s4) x iterations / kernel time; " +
                                 ("operators are staged in shared memory once per launch, so "
                                  "DRAM traffic is far below the algorithmic bytes"
                                  if info["sync"] != "stream-graph" else
                                  "operators are streamed from HBM every iteration")},
            "setup": {"partition": ("load-tuned CTA split of each scenario (dopf_cuda_tune_partition_batch on 74 "
                                    "scenarios, 6 rounds, untimed setup)" if batch else
                                    "tuned CTA split (dopf_cuda_tune_partition, 12 rounds, untimed setup; slack signal for grid-wide "
                                    "instances, load signal for cluster instances)")
                      if tuned_period else "default cost split"},
            "kernel": {"name": "admm_persistent" if info["sync"] != "stream-graph"
                       else "k_global+k_staged(+k_local), last chunk CTA folds + decides (graph while-node)",
                       "ctas_per_instance": info["blocks"],
                       "instances": info["instances"], "threads": info["threads"],
                       "smem_bytes": info["smem_bytes"], "resident": info["resident"],
                       "sync": info["sync"]},
            "clocks": clocks.summary(),
        }
        if batch:
            line["iterations_range"] = [int(min(last_its)), int(max(last_its))]
        if info["sync"] != "stream-graph":
            # the resident kernel reads its operators from shared memory every
            # iteration: the same algorithmic bytes against the SMs' aggregate
            # shared-memory bandwidth (128 B per cycle per SM at the sampled
            # clock), so a contract fraction near 1 is not read as HBM-bound
            mhz = line["clocks"].get("sm_mhz") or 1965.0
            sm = info.get("sm_count") or 148
            on_peak = sm * 128.0 * float(mhz) * 1e6 / 1e9
            line["roofline"]["onchip"] = {"bound": "smem", "achieved": achieved, "peak": on_peak, "unit": "GB/s",
                                          "frac": achieved / on_peak,
                                          "note": "148 SMs x 128 B/cycle x SM clock; DRAM traffic per launch is "
                                                  "the 'traffic' key"}
        if not args.no_cpu_baseline and world == 1:
            cores = os.cpu_count() or 1
            kw = dict(rho=100.0, eps_rel=1e-3)
            it_n = args.cpu_sample_iters or auto_cpu_iters(models, cores, kw)
            cps, cit, cdt, n = cpu_sample(models, kw, it_n, cores)
            what = (f"{it_n} ADMM iterations of each of {n} scenarios, one thread per scenario"
                    if n > 1 else f"{cit} ADMM iterations of the {args.config} solve, {cores} threads")
            # the same sample on ONE thread (workers = 1 figure), bounded to ~4 s
            one_n = max(5, int(it_n * min(1.0, 4.0 / max(cdt * cores, 1e-9)))) if n == 1 else it_n
            c1, c1it, c1dt, _ = cpu_sample(models[:1], kw, one_n, 1)
            line["cpu_baseline"] = {"value": cps, "unit": "iter/s", "cores": cores, "kind": "port",
                                    "cpu_model": cpu_model(),
                                    "value_1_thread": c1,
                                    "sample": f"{what} ({cdt:.1f} s, C++ oracle); 1-thread figure: {c1it} "
                                              f"iterations of one instance ({c1dt:.1f} s)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as td
        td.destroy_process_group()


if __name__ == "__main__":
    main()
