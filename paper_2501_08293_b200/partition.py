"""Partitioned solve of one large feeder over several ranks (one process per
GPU; BASELINE config 4: the tiled feeder split by subtree).

Each rank holds a contiguous, cost-balanced piece of the depth-first
component walk (for the tiled feeder: runs of whole tiles). Per iteration
(reference admm.cpp:190-235) every rank runs the HBM-streaming kernels on its
piece. The only exchange is one gather of the boundary copies' u = z -
lambda/rho (a few KB) plus 8 residual partials per rank. Every rank then sums
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
        self.model = model
        self.part_of_s = np.ascontiguousarray(
            partition_subsystems(model, self.world) if part_of_s is None else part_of_s, dtype=np.int32)
        self._err(self._lib.dopf_cuda_upload_part(self._h, C.byref(model.view()), self.world, self.rank,
                                                  self.part_of_s.ctypes.data_as(C.POINTER(N.i32))))
        info = N.PartInfo_t()
        self._err(self._lib.dopf_cuda_part_info(self._h, C.byref(info)))
        torch = self.torch
        dev = f"cuda:{self.device}"
        key = (info.send, info.recv, info.partials, info.ranks, info.max_export)
        # a captured graph bakes in the layout's kernel parameters (chunk
        # counts, boundary columns, export count): any upload invalidates it
        self._graph_key = None
        if getattr(self, "_buf_key", None) == key:
            self.info = info  # same buffers: the tensor views and the stream stay valid
            return
        self.info = info
        self._buf_key = key
        mx = max(1, info.max_export)
        self.send = torch.as_tensor(_DevArray(info.send, mx), device=dev)[:info.max_export]
        self.recv = torch.as_tensor(_DevArray(info.recv, max(1, self.world * info.max_export)),
                                    device=dev)[:self.world * info.max_export]
        self.partials = torch.as_tensor(_DevArray(info.partials, 8), device=dev)
        self.ranks = torch.as_tensor(_DevArray(info.ranks, 8 * self.world), device=dev)
        # one dedicated stream for the kernels AND the collectives (made current
        # around the loop), so they are ordered (a NULL handle would mean "own stream")
        if getattr(self, "stream", None) is None:
            self.stream = torch.cuda.Stream(device=dev)
            self._err(self._lib.dopf_cuda_set_stream(self._h, C.c_void_p(self.stream.cuda_stream)))
        self._graph_key = None
        # eager collective: communicator set-up must not happen inside a graph capture
        with torch.cuda.stream(self.stream):
            self._gather(self.ranks, self.partials)
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
        self._err(lib.dopf_cuda_part_step(h, 1))   # local, dual, exports, partials
        self._gather(self.recv, self.send)
        self._gather(self.ranks, self.partials)
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
                               tr[:it].copy() if trace else np.zeros((0, 6)), {"solve": r.time_solve},
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
