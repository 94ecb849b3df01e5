"""ctypes wrapper of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
--impl reference arm) import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2501_08293_b200 import _native as N
from paper_2501_08293_b200 import dopf

ORACLE_SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libdopf_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        N.host()
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle library missing: {ORACLE_SO}")
        L = C.CDLL(ORACLE_SO)
        P = C.POINTER
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_solve.restype = C.c_int
        L.oracle_solve.argtypes = [P(N.ModelView_t), P(N.Settings_t), P(N.ResultView_t),
                                   P(N.i32), N.i32, P(N.f64), P(N.f64), P(N.f64), P(N.f64)]
        L.oracle_reference_solve.restype = C.c_int
        L.oracle_reference_solve.argtypes = [P(N.LpView_t), N.i32, P(N.f64), P(N.f64), P(N.i32),
                                             P(N.f64), P(N.i32)]
        L.oracle_check_feasibility.restype = C.c_int
        L.oracle_check_feasibility.argtypes = [P(N.LpView_t), P(N.f64), P(N.f64), P(N.f64),
                                               P(N.i32), P(N.i32), P(N.f64)]
        L.oracle_reconstruct.restype = C.c_int
        L.oracle_reconstruct.argtypes = [P(N.ModelView_t), P(N.f64), P(N.f64), P(N.f64)]
        L.oracle_global_update.argtypes = [P(N.ModelView_t), P(N.f64), P(N.f64), N.f64, P(N.f64)]
        L.oracle_local_update.argtypes = [P(N.ModelView_t), N.i32, P(N.f64), P(N.f64), N.f64,
                                          P(N.f64)]
        L.oracle_dual_update.argtypes = [P(N.ModelView_t), N.i32, P(N.f64), P(N.f64), P(N.f64),
                                         N.f64]
        L.oracle_residuals.argtypes = [P(N.ModelView_t), P(N.f64), P(N.f64), P(N.f64), P(N.f64),
                                       N.f64, N.f64, P(N.f64)]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def solve(model: "dopf.DecomposedModel", settings: "dopf.Settings", snap_iters=()):
    """Restated reference solve loop (admm.cpp:172-244) on the CPU."""
    dopf._check_settings(settings)
    if not model.has_precompute:
        model.precompute(max(1, settings.workers))
    v = model.view()
    n, Nz = v.n, v.N_z
    x, z, lam = np.zeros(n), np.zeros(Nz), np.zeros(Nz)
    trace = np.zeros((settings.max_iter, 6))
    r = N.ResultView_t()
    r.x, r.z, r.lambda_, r.trace = _p(x), _p(z), _p(lam), _p(trace)
    snaps = np.array(sorted(snap_iters), dtype=np.int32)
    k = len(snaps)
    sx, sz, szp, sl = (np.zeros((max(k, 1), n)), np.zeros((max(k, 1), Nz)),
                       np.zeros((max(k, 1), Nz)), np.zeros((max(k, 1), Nz)))
    st = settings.to_c()
    rc = lib().oracle_solve(C.byref(v), C.byref(st), C.byref(r),
                            snaps.ctypes.data_as(C.POINTER(N.i32)), k,
                            _p(sx), _p(sz), _p(szp), _p(sl))
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)
    it = r.iterations
    res = dopf.SolveResult(x, z, lam, r.status, it, r.objective, r.max_local_infeasibility,
                           trace[:it].copy(), {"solve": r.time_solve, "global": r.time_global,
                                               "local": r.time_local, "dual": r.time_dual},
                           r.near_ties, r.first_near_tie)
    res.snapshots = {int(t): {"x": sx[i], "z": sz[i], "z_prev": szp[i], "lambda": sl[i]}
                     for i, t in enumerate(snaps) if t <= it}
    return res


def reference_solve(ls: "dopf.LinearSystem", max_cols: int = 500):
    """Dense two-phase simplex (oracle.cpp:164-273). Returns dict."""
    x = np.zeros(ls.cols)
    obj, kkt = C.c_double(), C.c_double()
    status, piv = N.i32(), N.i32()
    rc = lib().oracle_reference_solve(C.byref(ls.view), max_cols, _p(x), C.byref(obj),
                                      C.byref(status), C.byref(kkt), C.byref(piv))
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)
    return {"x": x, "objective": obj.value, "status": ["optimal", "infeasible", "unbounded"][status.value],
            "kkt_residual": kkt.value, "iterations": piv.value}


def check_feasibility(ls: "dopf.LinearSystem", x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (ls.cols,):
        raise ValueError(f"check_feasibility: x has {x.size} entries, model has {ls.cols} columns")
    eq, bd, obj = C.c_double(), C.c_double(), C.c_double()
    wr, wc = N.i32(), N.i32()
    lib().oracle_check_feasibility(C.byref(ls.view), _p(x), C.byref(eq), C.byref(bd),
                                   C.byref(wr), C.byref(wc), C.byref(obj))
    return {"max_equality_violation": eq.value, "max_bound_violation": bd.value,
            "worst_row": wr.value, "worst_col": wc.value, "objective": obj.value}


def reconstruct_centralized(model: "dopf.DecomposedModel", x, z):
    x = np.ascontiguousarray(x, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    out = np.zeros(model.global_cols)
    lib().oracle_reconstruct(C.byref(model.view()), _p(x), _p(z), _p(out))
    return out


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def global_update(model, z, lam, rho):
    """x from the copies (admm.cpp:118-129)."""
    x = np.zeros(model.global_cols)
    z, lam = _f(z), _f(lam)
    assert lib().oracle_global_update(C.byref(model.view()), _p(z), _p(lam), rho, _p(x)) == 0
    return x


def local_update(model, s, x, lam_s, rho):
    """z_s = P_s (x[l2g] + lambda_s / rho) + v_s (admm.cpp:131-138)."""
    zo = model.z_offsets
    out = np.zeros(int(zo[s + 1] - zo[s]))
    x, lam_s = _f(x), _f(lam_s)
    assert lib().oracle_local_update(C.byref(model.view()), s, _p(x), _p(lam_s), rho, _p(out)) == 0
    return out


def dual_update(model, s, x, z_s, lam_s, rho):
    """lambda_s + rho (x[l2g] - z_s) (admm.cpp:140-143); returns the new lambda_s."""
    lam = _f(lam_s).copy()
    x, z_s = _f(x), _f(z_s)
    assert lib().oracle_dual_update(C.byref(model.view()), s, _p(x), _p(z_s), _p(lam), rho) == 0
    return lam


def residuals(model, x, z, z_prev, lam, rho, eps_rel):
    """(pres, dres, eps_prim, eps_dual) (admm.cpp:145-170)."""
    out = np.zeros(4)
    x, z, z_prev, lam = _f(x), _f(z), _f(z_prev), _f(lam)
    assert lib().oracle_residuals(C.byref(model.view()), _p(x), _p(z), _p(z_prev), _p(lam), rho,
                                  eps_rel, _p(out)) == 0
    return tuple(float(v) for v in out)
