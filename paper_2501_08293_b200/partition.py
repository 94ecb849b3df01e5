"""Partitioned solve of one large feeder over several ranks (one process per
GPU; BASELINE config 4: the tiled feeder split by subtree).

Each rank holds a contiguous, cost-balanced piece of the depth-first
component walk (for the tiled feeder: runs of whole tiles). Per iteration
(reference admm.cpp:190-235) every rank runs the HBM-streaming kernels on its
piece. The only exchange is ONE gather per iteration of every rank's packed
record: the boundary copies' u = z - lambda/rho (a few KB) followed by its 8
residual partials. Every rank then sums
each boundary column's copies in ascending s, and combines the partials in
rank order, so iterates and the stop decision are bitwise identical on every
rank and equal to the single-GPU solve.

The collective is torch.distributed: NCCL on GPUs (CUDA tensors viewing the
solver's buffers, launched on the solver's stream), or gloo through host
copies (tests, several ranks sharing one GPU).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _native as N
from . import dopf


class _DevArray:
    """__cuda_array_interface__ view of solver-owned device memory (no copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def partition_subsystems(model: "dopf.DecomposedModel", nparts: int) -> np.ndarray:
    out = np.zeros(max(1, model.S), dtype=np.int32)
    rc = N.cuda().dopf_partition_subsystems(C.byref(model.view()), nparts,
                                           out.ctypes.data_as(C.POINTER(N.i32)))
    if rc != 0:
        raise RuntimeError("partition failed")
    return out[:model.S]


def probe_part(model, nparts: int, part: int, part_of_s: np.ndarray) -> dict:
    info = N.PartInfo_t()
    p = np.ascontiguousarray(part_of_s, dtype=np.int32)
    rc = N.cuda().dopf_layout_probe_part(C.byref(model.view()), nparts, part,
                                        p.ctypes.data_as(C.POINTER(N.i32)), C.byref(info))
    if rc != 0:
        raise ValueError("bad partition")
    return {"rows": info.rows, "cols": info.cols, "n_export": info.n_export,
            "max_export": info.max_export, "bytes_per_iteration": info.bytes_per_iteration}


def _partition_for(owner, model, nparts: int, part_of_s) -> np.ndarray:
    """The given map, else the cost-balanced walk partition -- computed once
    per model (a same-model re-upload, e.g. every e2e step, reuses it)."""
    if part_of_s is not None:
        return np.ascontiguousarray(part_of_s, dtype=np.int32)
    if getattr(owner, "model", None) is model and getattr(owner, "part_of_s", None) is not None:
        return owner.part_of_s
    return np.ascontiguousarray(partition_subsystems(model, nparts), dtype=np.int32)


class PartitionedSolver:
    """One rank's share of a partitioned solve (torch.distributed must be up)."""

    def __init__(self, device: int, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.device = device
        self.solver = dopf.CudaSolver(device)
        self._lib = self.solver._lib
        self._h = self.solver._h

    def _err(self, rc):
        self.solver._err(rc)

    def upload(self, model: "dopf.DecomposedModel", part_of_s: Optional[np.ndarray] = None):
        if not model.has_precompute:
            model.precompute()
        self.part_of_s = _partition_for(self, model, self.world, part_of_s)
        self.model = model
        self._err(self._lib.dopf_cuda_upload_part(self._h, C.byref(model.view()), self.world, self.rank,
                                                  self.part_of_s.ctypes.data_as(C.POINTER(N.i32))))
        info = N.PartInfo_t()
        self._err(self._lib.dopf_cuda_part_info(self._h, C.byref(info)))
        torch = self.torch
        dev = f"cuda:{self.device}"
        key = (info.send, info.recv, info.xstride)
        # a captured graph bakes in the layout's kernel parameters (chunk
        # counts, boundary columns, export count): any upload invalidates it
        self._graph_key = None
        if getattr(self, "_buf_key", None) == key:
            self.info = info  # same buffers: the tensor views and the stream stay valid
            return
        self.info = info
        self._buf_key = key
        # [exports | 8 partials] per rank, gathered in rank order
        self.send = torch.as_tensor(_DevArray(info.send, info.xstride), device=dev)
        self.recv = torch.as_tensor(_DevArray(info.recv, self.world * info.xstride), device=dev)
        # one dedicated stream for the kernels AND the collectives (made current
        # around the loop), so they are ordered (a NULL handle would mean "own stream")
        if getattr(self, "stream", None) is None:
            self.stream = torch.cuda.Stream(device=dev)
            self._err(self._lib.dopf_cuda_set_stream(self._h, C.c_void_p(self.stream.cuda_stream)))
        self._graph_key = None
        # eager collective: communicator set-up must not happen inside a graph capture
        with torch.cuda.stream(self.stream):
            self._gather(self.recv, self.send)
        self.stream.synchronize()

    def bytes_per_iteration(self) -> float:
        return float(self.info.bytes_per_iteration)

    def _gather(self, out, inp):
        if inp.numel() == 0:
            return
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        host = inp.cpu()
        parts = [self.torch.empty_like(host) for _ in range(self.world)]
        self.dist.all_gather(parts, host, group=self.group)
        out.copy_(self.torch.cat(parts).to(out.device))

    def solve(self, settings: "dopf.Settings", poll_every: int = 8, trace: bool = True,
              graph: "bool | None" = None):
        """Runs to the stop; returns this rank's share (x at owned columns, z /
        lambda at local rows) plus ownership masks. With NCCL the iteration
        (kernels + collectives) is captured once as a CUDA graph of
        `poll_every` iterations and replayed between stop checks."""
        dopf._check_settings(settings)
        if graph is None:
            graph = self.backend == "nccl"
        with self.torch.cuda.stream(self.stream):
            return self._solve(settings, poll_every, trace, graph)

    def _iteration(self):
        lib, h = self._lib, self._h
        self._err(lib.dopf_cuda_part_step(h, 0))   # global update (x^t)
        self._err(lib.dopf_cuda_part_step(h, 1))   # local, dual, exports + partials record
        self._gather(self.recv, self.send)          # the one exchange of the iteration
        self._err(lib.dopf_cuda_part_step(h, 2))   # identical stop decision everywhere

    def _solve(self, settings, poll_every, trace, graph):
        lib, h = self._lib, self._h
        st = settings.to_c()
        self._err(lib.dopf_cuda_part_begin(h, C.byref(st), 1 if trace else 0))
        self._err(lib.dopf_cuda_part_step(h, 3))       # exports of u^0
        self._gather(self.recv, self.send)
        done, its = N.i32(0), N.i32(0)
        key = (settings.rho, settings.eps_rel, settings.max_iter, trace, poll_every)
        if graph and getattr(self, "_graph_key", None) != key:
            # kernels after the stop are no-ops, so replaying whole chunks is exact
            g = self.torch.cuda.CUDAGraph()
            with self.torch.cuda.graph(g, stream=self.stream):
                for _ in range(poll_every):
                    self._iteration()
            self._graph, self._graph_key = g, key
            # capture only recorded the work: restart from iteration 0
            self._err(lib.dopf_cuda_part_begin(h, C.byref(st), 1 if trace else 0))
            self._err(lib.dopf_cuda_part_step(h, 3))
            self._gather(self.recv, self.send)
        k = 0
        while True:
            if graph:
                self._graph.replay()
                k += poll_every
            else:
                self._iteration()
                k += 1
            if k % poll_every == 0 or k >= settings.max_iter:
                self._err(lib.dopf_cuda_part_poll(h, C.byref(done), C.byref(its)))
                if done.value:
                    break
        return self._finish(settings, trace)

    def _finish(self, settings, trace):
        m = self.model
        n, Nz = m.global_cols, m.total_local_vars
        x, z, lam = np.zeros(n), np.zeros(Nz), np.zeros(Nz)
        xm, zm = np.zeros(n, dtype=np.uint8), np.zeros(Nz, dtype=np.uint8)
        tr = np.zeros((settings.max_iter, 6)) if trace else None
        r = N.ResultView_t()
        r.x = x.ctypes.data_as(C.POINTER(C.c_double))
        r.z = z.ctypes.data_as(C.POINTER(C.c_double))
        r.lambda_ = lam.ctypes.data_as(C.POINTER(C.c_double))
        if trace:
            r.trace = tr.ctypes.data_as(C.POINTER(C.c_double))
        self._err(self._lib.dopf_cuda_part_finish(self._h, C.byref(r), xm.ctypes.data_as(C.POINTER(C.c_uint8)),
                                                  zm.ctypes.data_as(C.POINTER(C.c_uint8))))
        it = r.iterations
        res = dopf.SolveResult(x, z, lam, r.status, it, r.objective, r.max_local_infeasibility,
                               tr[:it].copy() if trace else np.zeros((0, 6)), {"solve": r.time_solve, "global": r.time_global, "local": r.time_local,
                            "dual": r.time_dual},
                               r.near_ties, r.first_near_tie)
        res.x_mask, res.z_mask = xm.astype(bool), zm.astype(bool)
        return res

    def assemble(self, res) -> "dopf.SolveResult":
        """Whole-model x, z, lambda on every rank (each entry from its owner)."""
        objs = [None] * self.world
        self.dist.all_gather_object(objs, (res.x, res.x_mask, res.z, res.lam, res.z_mask), group=self.group)
        x, z, lam = np.zeros_like(res.x), np.zeros_like(res.z), np.zeros_like(res.lam)
        xs, zs = np.zeros(len(x), dtype=int), np.zeros(len(z), dtype=int)
        for (px, pxm, pz, pl, pzm) in objs:
            x[pxm], z[pzm], lam[pzm] = px[pxm], pz[pzm], pl[pzm]
            xs += pxm
            zs += pzm
        if not (np.all(xs == 1) and np.all(zs == 1)):
            raise RuntimeError("partition does not cover every column / copy exactly once")
        return dopf.SolveResult(x, z, lam, res.status, res.iterations, res.objective,
                                res.max_local_infeasibility, res.trace, res.timings, res.near_ties,
                                res.first_near_tie)


# --------------------------------------------------------------------------
# The library's own NCCL path (C ABI dopf_cuda_comm_init / dopf_cuda_solve_part):
# the whole partitioned loop -- kernels and one ncclAllGather of the packed
# records per iteration -- is one CUDA graph on the device; Python only sets
# it up. torch.distributed (any backend) carries the 128-byte NCCL id.


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = N.cuda().dopf_nccl_unique_id(buf)
    if rc != 0:
        raise RuntimeError("ncclGetUniqueId failed: " + (N.cuda().dopf_nccl_describe() or b"").decode())
    return buf.raw


def _share_of(solver: "dopf.CudaSolver", model, settings, trace):
    n, Nz = model.global_cols, model.total_local_vars
    x, z, lam = np.zeros(n), np.zeros(Nz), np.zeros(Nz)
    xm, zm = np.zeros(n, dtype=np.uint8), np.zeros(Nz, dtype=np.uint8)
    tr = np.zeros((settings.max_iter, 6)) if trace else None
    r = N.ResultView_t()
    r.x = x.ctypes.data_as(C.POINTER(C.c_double))
    r.z = z.ctypes.data_as(C.POINTER(C.c_double))
    r.lambda_ = lam.ctypes.data_as(C.POINTER(C.c_double))
    if trace:
        r.trace = tr.ctypes.data_as(C.POINTER(C.c_double))
    st = settings.to_c()
    rc = solver._lib.dopf_cuda_solve_part(solver._h, C.byref(st), C.byref(r),
                                          xm.ctypes.data_as(C.POINTER(C.c_uint8)),
                                          zm.ctypes.data_as(C.POINTER(C.c_uint8)))
    return rc, r, (x, z, lam, xm, zm, tr)


def _result(r, bufs):
    x, z, lam, xm, zm, tr = bufs
    it = r.iterations
    res = dopf.SolveResult(x, z, lam, r.status, it, r.objective, r.max_local_infeasibility,
                           tr[:it].copy() if tr is not None else np.zeros((0, 6)), {"solve": r.time_solve, "global": r.time_global, "local": r.time_local,
                            "dual": r.time_dual},
                           r.near_ties, r.first_near_tie)
    res.x_mask, res.z_mask = xm.astype(bool), zm.astype(bool)
    return res


def merge_shares(shares) -> "dopf.SolveResult":
    """Whole-model x, z, lambda from every rank's share (each entry from its
    owner); scalars and trace are identical on every rank."""
    first = shares[0]
    x, z, lam = np.zeros_like(first.x), np.zeros_like(first.z), np.zeros_like(first.lam)
    xs, zs = np.zeros(len(x), dtype=int), np.zeros(len(z), dtype=int)
    for s in shares:
        x[s.x_mask], z[s.z_mask], lam[s.z_mask] = s.x[s.x_mask], s.z[s.z_mask], s.lam[s.z_mask]
        xs += s.x_mask
        zs += s.z_mask
    if not (np.all(xs == 1) and np.all(zs == 1)):
        raise RuntimeError("partition does not cover every column / copy exactly once")
    return dopf.SolveResult(x, z, lam, first.status, first.iterations, first.objective,
                            first.max_local_infeasibility, first.trace, first.timings, first.near_ties,
                            first.first_near_tie)


class NcclPartitionedSolver:
    """One rank (one process, one GPU) of a partitioned solve on the
    library's NCCL communicator. `unique_id` comes from nccl_unique_id() on
    rank 0, shared by the caller (see from_torch_distributed)."""

    def __init__(self, device: int, nranks: int, rank: int, unique_id: bytes):
        self.solver = dopf.CudaSolver(device)
        self.nranks, self.rank = nranks, rank
        self.solver._err(self.solver._lib.dopf_cuda_comm_init(self.solver._h, nranks, rank, unique_id))

    @classmethod
    def from_torch_distributed(cls, device: int, group=None) -> "NcclPartitionedSolver":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        return cls(device, world, rank, box[0])

    def upload(self, model: "dopf.DecomposedModel", part_of_s: Optional[np.ndarray] = None):
        if not model.has_precompute:
            model.precompute()
        self.part_of_s = _partition_for(self, model, self.nranks, part_of_s)
        self.model = model
        s = self.solver
        s._err(s._lib.dopf_cuda_upload_part(s._h, C.byref(model.view()), self.nranks, self.rank,
                                            self.part_of_s.ctypes.data_as(C.POINTER(N.i32))))
        s.model = model

    def solve(self, settings: "dopf.Settings", trace: bool = True) -> "dopf.SolveResult":
        dopf._check_settings(settings)
        rc, r, bufs = _share_of(self.solver, self.model, settings, trace)
        self.solver._err(rc)
        return _result(r, bufs)

    def graph_mode(self) -> str:
        return {0: "none", 1: "while-node", 2: "unrolled"}[self.solver._lib.dopf_cuda_part_graph_mode(self.solver._h)]

    def bytes_per_iteration(self) -> float:
        return self.solver.bytes_per_iteration()

    def last_kernel_seconds(self) -> float:
        return float(self.solver._lib.dopf_cuda_last_kernel_seconds(self.solver._h))


class MultiGpuSolver:
    """One process driving n GPUs (one context each, ncclCommInitAll): the
    partitioned solve of one model, the ranks' loops on threads (the C ABI
    releases the GIL)."""

    def __init__(self, devices):
        self.devices = list(devices)
        self.solvers = [dopf.CudaSolver(d) for d in self.devices]
        arr = (C.c_void_p * len(self.solvers))(*[s._h.value for s in self.solvers])
        self.solvers[0]._err(self.solvers[0]._lib.dopf_cuda_comm_init_all(arr, len(self.solvers)))

    def upload(self, model: "dopf.DecomposedModel", part_of_s: Optional[np.ndarray] = None):
        if not model.has_precompute:
            model.precompute()
        n = len(self.solvers)
        self.model = model
        self.part_of_s = np.ascontiguousarray(
            partition_subsystems(model, n) if part_of_s is None else part_of_s, dtype=np.int32)
        for k, s in enumerate(self.solvers):
            s._err(s._lib.dopf_cuda_upload_part(s._h, C.byref(model.view()), n, k,
                                                self.part_of_s.ctypes.data_as(C.POINTER(N.i32))))
            s.model = model

    def solve(self, settings: "dopf.Settings", trace: bool = True) -> "dopf.SolveResult":
        import concurrent.futures as cf
        dopf._check_settings(settings)
        with cf.ThreadPoolExecutor(max_workers=len(self.solvers)) as ex:
            outs = list(ex.map(lambda s: _share_of(s, self.model, settings, trace), self.solvers))
        shares = []
        for s, (rc, r, bufs) in zip(self.solvers, outs):
            s._err(rc)
            shares.append(_result(r, bufs))
        return merge_shares(shares)
