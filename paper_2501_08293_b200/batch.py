"""Independent load scenarios solved together (BASELINE config 5).

Each scenario is an independent reference `solve` (own iteration count and
trace, admm.cpp:172-244); on the device each runs on its own cluster of CTAs
and stops at its own convergence iteration.
"""
from __future__ import annotations

import ctypes as C
from typing import List

import numpy as np

from . import _native as N
from . import dopf


class BatchSolver:
    def __init__(self, device: int = 0):
        self._s = dopf.CudaSolver(device)
        self.models: List[dopf.DecomposedModel] = []

    def upload(self, models: List[dopf.DecomposedModel]) -> None:
        for m in models:
            if not m.has_precompute:
                m.precompute()
        views = (N.ModelView_t * len(models))(*[m.view() for m in models])
        self._s._err(self._s._lib.dopf_cuda_upload_batch(self._s._h, views, len(models)))
        self.models = list(models)
        self._views = views

    def tune_partition(self, models: List[dopf.DecomposedModel], settings: dopf.Settings = None,
                       rounds: int = 6) -> float:
        """Setup-time tuning of one instance's CTA split on a sample of the
        scenarios (dopf_cuda_tune_partition_batch); the next upload of this
        structure keeps it. Returns seconds per scenario-iteration."""
        for m in models:
            if not m.has_precompute:
                m.precompute()
        views = (N.ModelView_t * len(models))(*[m.view() for m in models])
        st = (settings or dopf.Settings()).to_c()
        out = C.c_double(0.0)
        self._s._err(self._s._lib.dopf_cuda_tune_partition_batch(self._s._h, views, len(models), C.byref(st),
                                                                 rounds, C.byref(out)))
        return out.value

    def info(self) -> dict:
        return self._s.info()

    def kernel_launches(self) -> int:
        return self._s.kernel_launches()

    def bytes_per_iteration(self) -> float:
        return self._s.bytes_per_iteration()

    def solve(self, settings: dopf.Settings, outputs: bool = True, trace: bool = True):
        dopf._check_settings(settings)
        k = len(self.models)
        rs = (N.ResultView_t * k)()
        bufs = []
        for i, m in enumerate(self.models):
            v = m.view()
            x, z, lam = np.zeros(v.n), np.zeros(v.N_z), np.zeros(v.N_z)
            tr = np.zeros((settings.max_iter, 6)) if trace else None
            if outputs:
                rs[i].x = x.ctypes.data_as(C.POINTER(C.c_double))
                rs[i].z = z.ctypes.data_as(C.POINTER(C.c_double))
                rs[i].lambda_ = lam.ctypes.data_as(C.POINTER(C.c_double))
            if trace:
                rs[i].trace = tr.ctypes.data_as(C.POINTER(C.c_double))
            bufs.append((x, z, lam, tr))
        st = settings.to_c()
        self._s._err(self._s._lib.dopf_cuda_solve_batch(self._s._h, C.byref(st), rs, k))
        out = []
        for i in range(k):
            x, z, lam, tr = bufs[i]
            it = rs[i].iterations
            out.append(dopf.SolveResult(x, z, lam, rs[i].status, it, rs[i].objective,
                                        rs[i].max_local_infeasibility,
                                        tr[:it].copy() if tr is not None else np.zeros((0, 6)),
                                        {"solve": rs[i].time_solve, "global": rs[i].time_global,
                                         "local": rs[i].time_local, "dual": rs[i].time_dual}, rs[i].near_ties,
                                        rs[i].first_near_tie))
        return out
