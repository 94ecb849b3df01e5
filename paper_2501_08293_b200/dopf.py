"""Python mirror of the reference's `dopf` C++ API for the ADMM hot path.

Names, argument meaning and error behaviour follow the reference headers:
  parse_feeder / parse_feeder_file / validate_feeder / serialize_feeder
      proj/include/dopf/feeder.hpp:112-124
  assemble_centralized                  proj/include/dopf/lp_builder.hpp:57
  decompose / partition / reduce_subsystems
      proj/include/dopf/decompose.hpp:84-91
  Settings, precompute, solve, SolveResult, TraceRow, write_trace_csv,
  write_solution                        proj/include/dopf/admm.hpp:14-133
`solve` runs the iteration on the GPU (sm_100a kernels behind
include/dopf_cuda.h); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N

# ---------------------------------------------------------------- errors


class ParseError(RuntimeError):
    pass


class SingularSubsystemError(RuntimeError):
    def __init__(self, msg: str):
        super().__init__(msg)
        # "numerically singular subsystem '<id>'"
        self.subsystem_id = msg.split("'")[1] if "'" in msg else ""


class InfeasibleSubsystemError(RuntimeError):
    def __init__(self, msg: str):
        super().__init__(msg)
        self.subsystem_id = msg.split("'")[1] if "'" in msg else ""


class CudaError(RuntimeError):
    pass


def _raise(code: int, msg: str):
    if code == 0:
        return
    if code == 1:
        raise ValueError(msg)          # std::invalid_argument
    if code == 2:
        raise SingularSubsystemError(msg)
    if code in (3, 4):
        raise CudaError(msg)
    if code == 5:
        raise MemoryError(msg)
    if code == 6:
        raise ParseError(msg)
    if code == 7:
        raise InfeasibleSubsystemError(msg)
    if code == 8:
        raise AssertionError(msg)      # std::logic_error
    raise RuntimeError(msg)


def _release(obj, free_name: str, _native=N) -> None:
    """Frees a native handle once. Safe during interpreter shutdown, when
    module globals (the native library bindings) may already be gone."""
    h = getattr(obj, "_h", None)
    obj._h = None
    if h is None or not h.value:
        return
    try:
        getattr(_native.host(), free_name)(h)
    except Exception:  # shutdown: the process is exiting, the OS reclaims it
        pass


def _check(code: int):
    if code != 0:
        _raise(code, N.last_error())


# ---------------------------------------------------------------- feeder


@dataclass
class Diagnostic:
    severity: str
    component: str
    message: str


class Feeder:
    """Owning handle of a parsed, id-sorted feeder (reference Feeder)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self, _rel=_release):  # bound at definition: module globals are gone at shutdown
        _rel(self, "dopf_feeder_free")

    @property
    def handle(self):
        return self._h

    def counts(self) -> dict:
        out = (N.i32 * 5)()
        _check(N.host().dopf_feeder_counts(self._h, out))
        return {"buses": out[0], "generators": out[1], "lines": out[2], "loads": out[3],
                "leaves": out[4]}

    def serialize(self) -> str:
        rc, text = N.text_call(N.host().dopf_feeder_serialize, self._h)
        _check(rc)
        return text


def _new_feeder(fn, *args) -> Feeder:
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)))
    return Feeder(h.value)


def parse_feeder(text: str) -> Feeder:
    raw = text.encode()
    return _new_feeder(N.host().dopf_feeder_parse, raw, len(raw))


def parse_feeder_file(path: str) -> Feeder:
    return _new_feeder(N.host().dopf_feeder_parse_file, str(path).encode())


def synthetic_feeder(shape: str, seed: int) -> Feeder:
    """Seeded feeder with the paper's structural counts ("ieee13"/"ieee123"/"ieee8500")."""
    return _new_feeder(N.host().dopf_feeder_synthetic, shape.encode(), seed)


def tiled_feeder(shape: str, copies: int, seed: int) -> Feeder:
    return _new_feeder(N.host().dopf_feeder_synthetic_tiled, shape.encode(), copies, seed)


def scale_loads(base: Feeder, seed: int) -> Feeder:
    return _new_feeder(N.host().dopf_feeder_scale_loads, base.handle, seed)


def serialize_feeder(f: Feeder) -> str:
    return f.serialize()


def validate_feeder(f: Feeder) -> List[Diagnostic]:
    n_err = N.i32(0)
    need = N.sz(0)
    lib = N.host()
    _check(lib.dopf_feeder_validate(f.handle, None, 0, C.byref(need), C.byref(n_err)))
    buf = C.create_string_buffer(need.value)
    _check(lib.dopf_feeder_validate(f.handle, buf, need.value, C.byref(need), C.byref(n_err)))
    diags = []
    for line in buf.value.decode().splitlines():
        sev, comp, msg = line.split("\t", 2)
        diags.append(Diagnostic(sev, comp, msg))
    return diags


def has_errors(diags: List[Diagnostic]) -> bool:
    return any(d.severity == "error" for d in diags)


# ---------------------------------------------------------------- LP


VAR_KINDS = ["p_gen", "q_gen", "w", "p_bus_load", "q_bus_load", "p_load", "q_load", "p_flow",
             "q_flow"]


class LinearSystem:
    """Centralized LP min c'x, Ax=b, lo<=x<=hi (reference LinearSystem)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        v = N.LpView_t()
        _check(N.host().dopf_lp_view_get(self._h, C.byref(v)))
        self._v = v
        self.rows, self.cols, self.nnz = v.rows, v.cols, v.nnz

    def __del__(self, _rel=_release):  # bound at definition: module globals are gone at shutdown
        _rel(self, "dopf_lp_free")

    @property
    def handle(self):
        return self._h

    @property
    def view(self) -> N.LpView_t:
        return self._v

    def _arr(self, ptr, n):
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n else np.zeros(0)

    @property
    def row_ptr(self):
        return self._arr(self._v.row_ptr, self.rows + 1)

    @property
    def col_idx(self):
        return self._arr(self._v.col_idx, self.nnz)

    @property
    def values(self):
        return self._arr(self._v.values, self.nnz)

    @property
    def b(self):
        return self._arr(self._v.b, self.rows)

    @property
    def c(self):
        return self._arr(self._v.c, self.cols)

    @property
    def x_lo(self):
        return self._arr(self._v.x_lo, self.cols)

    @property
    def x_hi(self):
        return self._arr(self._v.x_hi, self.cols)

    @property
    def var_kind(self):
        return self._arr(self._v.var_kind, self.cols)

    def dense(self) -> np.ndarray:
        a = np.zeros((self.rows, self.cols))
        rp, ci, vals = self.row_ptr, self.col_idx, self.values
        for i in range(self.rows):
            a[i, ci[rp[i]:rp[i + 1]]] = vals[rp[i]:rp[i + 1]]
        return a

    def var_key(self, col: int) -> str:
        buf = C.create_string_buffer(512)
        _check(N.host().dopf_lp_var_key(self._h, col, buf, 512))
        return buf.value.decode()

    def row_tag(self, row: int) -> str:
        buf = C.create_string_buffer(512)
        _check(N.host().dopf_lp_row_tag(self._h, row, buf, 512))
        return buf.value.decode()

    def var_table(self) -> List[str]:
        return [self.var_key(j) for j in range(self.cols)]

    def column(self, key: str) -> int:
        for j in range(self.cols):
            if self.var_key(j) == key:
                return j
        raise KeyError(key)

    def dump(self) -> str:
        rc, text = N.text_call(N.host().dopf_lp_dump, self._h)
        _check(rc)
        return text


LOAD_KINDS = {"constant_power": 0, "constant_current": 1, "constant_impedance": 2}


def derive_load_coefficients(p_ref: float, q_ref: float, kind: str) -> dict:
    """Reference derive_load_coefficients (feeder.hpp:104-110)."""
    out = (C.c_double * 4)()
    _check(N.host().dopf_derive_load_coefficients(p_ref, q_ref, LOAD_KINDS[kind], out))
    return {"a": out[0], "b": out[1], "alpha": out[2], "beta": out[3]}


def line_m_matrices(phases, r, x):
    """Reference build_m_matrices (lp_builder.cpp:275-296) of one line."""
    ph = np.ascontiguousarray(phases, dtype=np.int32)
    n = len(ph)
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(n, n)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(n, n)
    mp, mq = np.zeros((n, n)), np.zeros((n, n))
    dp = C.POINTER(C.c_double)
    _check(N.host().dopf_line_m_matrices(n, ph.ctypes.data_as(C.POINTER(N.i32)), r.ctypes.data_as(dp),
                                         x.ctypes.data_as(dp), mp.ctypes.data_as(dp), mq.ctypes.data_as(dp)))
    return mp, mq


def assemble_centralized(f: Feeder) -> LinearSystem:
    h = C.c_void_p()
    _check(N.host().dopf_lp_assemble(f.handle, C.byref(h)))
    return LinearSystem(h.value)


# ---------------------------------------------------------------- decomposed model


@dataclass
class Settings:
    rho: float = 100.0
    eps_rel: float = 1e-3
    max_iter: int = 50000
    workers: int = 1
    record_iterates: bool = False

    def to_c(self) -> N.Settings_t:
        return N.Settings_t(float(self.rho), float(self.eps_rel), int(self.max_iter),
                            int(self.workers), int(bool(self.record_iterates)), 0)


class DecomposedModel:
    """Decomposed model + (after precompute) the per-subsystem operators."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self._view: Optional[N.ModelView_t] = None

    def __del__(self, _rel=_release):  # bound at definition: module globals are gone at shutdown
        _rel(self, "dopf_model_free")

    @property
    def handle(self):
        return self._h

    def view(self) -> N.ModelView_t:
        if self._view is None:
            v = N.ModelView_t()
            _check(N.host().dopf_model_view_get(self._h, C.byref(v)))
            self._view = v
        return self._view

    def precompute(self, workers: int = 1) -> "DecomposedModel":
        """One-time operators P_s, v_s (reference admm.cpp:31-88)."""
        _check(N.host().dopf_model_precompute(self._h, workers))
        self._view = None
        return self

    def precompute_gpu(self, solver: "CudaSolver") -> "DecomposedModel":
        """One-time operators on the GPU (batched kernel, bitwise equal to precompute())."""
        v = self.view()
        S = v.S
        zo = np.ctypeslib.as_array(v.z_offsets, shape=(S + 1,)) if S else np.zeros(1, dtype=np.int32)
        ns = np.diff(zo).astype(np.int64)
        P = np.zeros(int((ns * ns).sum()))
        vv = np.zeros(int(v.N_z))
        first = N.i32(-1)
        rc = solver._lib.dopf_cuda_precompute(solver._h, C.byref(v), P.ctypes.data_as(C.POINTER(C.c_double)),
                                              vv.ctypes.data_as(C.POINTER(C.c_double)), C.byref(first))
        if rc == 2 and first.value >= 0:
            raise SingularSubsystemError(f"numerically singular subsystem '{self.component_id(first.value)}'")
        solver._err(rc)
        _check(N.host().dopf_model_set_operators(self._h, P.ctypes.data_as(C.POINTER(C.c_double)),
                                                 vv.ctypes.data_as(C.POINTER(C.c_double))))
        self._view = None
        return self

    def reduce(self, tol: float = 1e-9, workers: int = 1) -> None:
        _check(N.host().dopf_model_reduce(self._h, tol, workers))
        self._view = None

    @property
    def has_precompute(self) -> bool:
        return bool(self.view().has_pre)

    @property
    def S(self) -> int:
        return self.view().S

    @property
    def global_cols(self) -> int:
        return self.view().n

    @property
    def total_local_vars(self) -> int:
        return self.view().N_z

    def arr(self, name: str) -> np.ndarray:
        v = self.view()
        S, n, Nz = v.S, v.n, v.N_z
        sizes = {"z_offsets": S + 1, "l2g": Nz, "m_s": S, "a_offsets": S + 1,
                 "b_offsets": S + 1, "p_offsets": S + 1, "v": Nz, "inv_copy": n,
                 "csr_ptr": n + 1, "csr_copy": Nz, "c": n, "x_lo": n, "x_hi": n, "x0": n,
                 "z0": Nz}
        if name == "A":
            size = int(self.arr("a_offsets")[-1])
        elif name == "b":
            size = int(self.arr("b_offsets")[-1])
        elif name == "P":
            size = int(self.arr("p_offsets")[-1])
        else:
            size = sizes[name]
        ptr = getattr(v, name)
        if not ptr or size == 0:
            return np.zeros(size)
        return np.ctypeslib.as_array(ptr, shape=(size,)).copy()

    @property
    def z_offsets(self):
        return self.arr("z_offsets")

    @property
    def copy_counts(self):
        return np.diff(self.arr("csr_ptr")) if self.has_precompute else \
            np.bincount(self.arr("l2g"), minlength=self.global_cols)

    def subsystem(self, s: int) -> dict:
        zo = self.arr("z_offsets")
        ao = self.arr("a_offsets")
        bo = self.arr("b_offsets")
        ns = int(zo[s + 1] - zo[s])
        ms = int(self.arr("m_s")[s])
        out = {"component_id": self.component_id(s),
               "A": self.arr("A")[ao[s]:ao[s + 1]].reshape(ms, ns),
               "b": self.arr("b")[bo[s]:bo[s + 1]],
               "local_to_global": self.arr("l2g")[zo[s]:zo[s + 1]]}
        if self.has_precompute:
            po = self.arr("p_offsets")
            out["P"] = self.arr("P")[po[s]:po[s + 1]].reshape(ns, ns)
            out["v"] = self.arr("v")[zo[s]:zo[s + 1]]
        return out

    def component_id(self, s: int) -> str:
        buf = C.create_string_buffer(1024)
        _check(N.host().dopf_model_component_id(self._h, s, buf, 1024))
        return buf.value.decode()

    def rows_before_reduction(self) -> np.ndarray:
        out = (N.i32 * max(1, self.S))()
        _check(N.host().dopf_model_rows_before_reduction(self._h, out))
        return np.array(out[:self.S], dtype=np.int32)

    def dump_subsystems(self) -> str:
        rc, text = N.text_call(N.host().dopf_model_dump_subsystems, self._h)
        _check(rc)
        return text

    def stats(self) -> dict:
        zo = self.arr("z_offsets")
        ns = np.diff(zo)
        ms = self.arr("m_s")
        return {"S": int(self.S), "n": int(self.global_cols), "N_z": int(zo[-1]),
                "sum_m": int(ms.sum()), "sum_n2": int((ns.astype(np.int64) ** 2).sum()),
                "sum_mn": int((ms.astype(np.int64) * ns).sum()),
                "m_mean": float(ms.mean()) if len(ms) else 0.0,
                "m_max": int(ms.max()) if len(ms) else 0,
                "n_mean": float(ns.mean()) if len(ns) else 0.0,
                "n_max": int(ns.max()) if len(ns) else 0,
                "n_min": int(ns.min()) if len(ns) else 0,
                "n_std": float(ns.std()) if len(ns) else 0.0,
                "m_std": float(ms.std()) if len(ms) else 0.0}


def decompose(ls: LinearSystem, f: Feeder, tol: float = 1e-9, workers: int = 1) -> DecomposedModel:
    h = C.c_void_p()
    _check(N.host().dopf_model_decompose(ls.handle, f.handle, tol, workers, C.byref(h)))
    return DecomposedModel(h.value)


def partition(ls: LinearSystem, f: Feeder) -> DecomposedModel:
    h = C.c_void_p()
    _check(N.host().dopf_model_partition(ls.handle, f.handle, C.byref(h)))
    return DecomposedModel(h.value)


def prepare_gpu(models: List["DecomposedModel"], solver: "CudaSolver", tol: float = 1e-9,
                chunk: int = 512) -> dict:
    """GPU equivalent of ``m.reduce(tol); m.precompute()`` for every model
    (SURVEY row f2): row_reduce (reference decompose.cpp:48-98) and the
    operators (admm.cpp:31-88) of all subsystems of `chunk` models per pair of
    launches (dopf_cuda_prepare), bitwise equal to the host. `models` are
    partitioned, unreduced models. Raises InfeasibleSubsystemError /
    SingularSubsystemError naming the component like the host does. Returns
    the summed {pack, kernels, unpack} seconds of the device calls."""
    import concurrent.futures as cf
    import os
    tot = {"pack_s": 0.0, "kernels_s": 0.0, "unpack_s": 0.0}
    # per-model host bookkeeping (views, adopting the results) on all cores:
    # ctypes releases the GIL inside the native calls
    pool = cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 1)
    for c0 in range(0, len(models), chunk):
        part = models[c0:c0 + chunk]
        views = (N.ModelView_t * len(part))(*pool.map(lambda m: m.view(), part))
        na = nb = ns = npp = nz = 0
        sizes = []
        for v in views:
            S = v.S
            a = int(v.a_offsets[S]) if S else 0
            b = int(v.b_offsets[S]) if S else 0
            zo = np.ctypeslib.as_array(v.z_offsets, shape=(S + 1,)) if S else np.zeros(1, np.int32)
            p2 = int((np.diff(zo).astype(np.int64) ** 2).sum())
            sizes.append((a, b, S, p2, int(v.N_z)))
            na, nb, ns, npp, nz = na + a, nb + b, ns + S, npp + p2, nz + int(v.N_z)
        A, B = np.zeros(max(na, 1)), np.zeros(max(nb, 1))
        Ms = np.zeros(max(ns, 1), dtype=np.int32)
        Pp, V = np.zeros(max(npp, 1)), np.zeros(max(nz, 1))
        out = N.PrepareOut_t(A.ctypes.data_as(C.POINTER(C.c_double)), B.ctypes.data_as(C.POINTER(C.c_double)),
                             Ms.ctypes.data_as(C.POINTER(N.i32)), Pp.ctypes.data_as(C.POINTER(C.c_double)),
                             V.ctypes.data_as(C.POINTER(C.c_double)))
        fm, fs = N.i32(-1), N.i32(-1)
        secs = (C.c_double * 3)()
        rc = solver._lib.dopf_cuda_prepare(solver._h, views, len(part), tol, C.byref(out), C.byref(fm),
                                           C.byref(fs), secs)
        if rc == 7:
            raise InfeasibleSubsystemError(
                f"infeasible subsystem '{part[fm.value].component_id(fs.value)}': contradictory rows")
        if rc == 2:
            raise SingularSubsystemError(
                f"numerically singular subsystem '{part[fm.value].component_id(fs.value)}'")
        solver._err(rc)
        tot["pack_s"] += secs[0]
        tot["kernels_s"] += secs[1]
        tot["unpack_s"] += secs[2]
        starts, a0 = [], (0, 0, 0, 0, 0)
        for (a, b, S, p2, n_z) in sizes:
            starts.append(a0)
            a0 = (a0[0] + a, a0[1] + b, a0[2] + S, a0[3] + p2, a0[4] + n_z)
        dp, ip = C.POINTER(C.c_double), C.POINTER(N.i32)
        base = (A.ctypes.data, B.ctypes.data, Ms.ctypes.data, Pp.ctypes.data, V.ctypes.data)

        def adopt(job):
            m, (oa, ob, os_, op, oz) = job
            _check(N.host().dopf_model_set_reduced(m.handle, C.cast(base[0] + 8 * oa, dp),
                                                   C.cast(base[1] + 8 * ob, dp), C.cast(base[2] + 4 * os_, ip)))
            _check(N.host().dopf_model_set_operators(m.handle, C.cast(base[3] + 8 * op, dp),
                                                     C.cast(base[4] + 8 * oz, dp)))
            m._view = None

        list(pool.map(adopt, zip(part, starts)))
    pool.shutdown()
    return tot


def model_from_arrays(subsystems, c, x_lo, x_hi, is_w=None) -> DecomposedModel:
    """Build a model from dense subsystem data.

    subsystems: list of (A (m x n_s), b (m), local_to_global (n_s)).
    Mirrors test_util.hpp:52-74 (single_sub_model) and the hand-built
    multi-copy models of test_admm.cpp:113-173.
    """
    n = len(c)
    z_off = [0]
    l2g, ms, A, b = [], [], [], []
    for (a, bb, cols) in subsystems:
        a = np.asarray(a, dtype=np.float64).reshape(len(bb), len(cols))
        z_off.append(z_off[-1] + len(cols))
        l2g += list(cols)
        ms.append(a.shape[0])
        A += list(a.reshape(-1))
        b += list(np.asarray(bb, dtype=np.float64))

    def arr(t, xs):
        xs = list(xs)
        return (t * max(1, len(xs)))(*xs)

    isw = arr(N.i32, [int(v) for v in (is_w if is_w is not None else [0] * n)])
    h = C.c_void_p()
    _check(N.host().dopf_model_from_arrays(
        len(subsystems), n, arr(N.i32, z_off), arr(N.i32, l2g), arr(N.i32, ms), arr(N.f64, A),
        arr(N.f64, b), arr(N.f64, c), arr(N.f64, x_lo), arr(N.f64, x_hi), isw, C.byref(h)))
    return DecomposedModel(h.value)


def single_sub_model(a, b, c, lo, hi) -> DecomposedModel:
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[1]
    return model_from_arrays([(a, b, list(range(n)))], c, lo, hi)


# ---------------------------------------------------------------- results + solve


CONVERGED, ITERATION_LIMIT = 0, 1


@dataclass
class TraceRow:
    t: int
    pres: float
    dres: float
    eps_prim: float
    eps_dual: float
    objective: float


@dataclass
class SolveResult:
    x: np.ndarray
    z: np.ndarray
    lam: np.ndarray
    status: int
    iterations: int
    objective: float
    max_local_infeasibility: float
    trace: np.ndarray            # (iterations, 6): t, pres, dres, eps_prim, eps_dual, objective
    timings: dict = field(default_factory=dict)
    # stop tests within 1e-12 relative of flipping (dopf_result_view.near_ties)
    near_ties: int = 0
    first_near_tie: int = 0
    # parity mode: t -> {x, z, z_prev, lambda} after iteration t (CudaSolver.solve(snapshots=T))
    snapshots: dict = field(default_factory=dict)

    @property
    def converged(self) -> bool:
        return self.status == CONVERGED

    def trace_rows(self) -> List[TraceRow]:
        return [TraceRow(int(r[0]), *map(float, r[1:])) for r in self.trace]


def _check_settings(settings: Settings):
    # reference admm.cpp:173-175
    if not settings.rho > 0:
        raise ValueError("rho must be positive")
    if not settings.eps_rel > 0:
        raise ValueError("eps_rel must be positive")
    if settings.max_iter < 1:
        raise ValueError("max_iter must be positive")


class CudaSolver:
    """One device context: uploads a model once, solves many times."""

    def __init__(self, device: int = 0):
        lib = N.cuda()
        h = C.c_void_p()
        rc = lib.dopf_cuda_create(device, C.byref(h))
        if rc != 0:
            _raise(rc, "dopf_cuda_create failed: " + (N.last_error() or "no CUDA device"))
        self._h = h
        self._lib = lib
        self.model: Optional[DecomposedModel] = None

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        lib = getattr(self, "_lib", None)
        if h is not None and h.value and lib is not None:
            try:
                lib.dopf_cuda_destroy(h)
            except Exception:  # interpreter shutdown
                pass

    def _err(self, rc):
        if rc != 0:
            msg = self._lib.dopf_cuda_last_error(self._h)
            _raise(rc, msg.decode() if msg else "CUDA solver error")

    def upload(self, model: DecomposedModel) -> None:
        if not model.has_precompute:
            model.precompute()
        self._err(self._lib.dopf_cuda_upload(self._h, C.byref(model.view())))
        self.model = model

    def info(self) -> dict:
        i = N.BatchInfo_t()
        self._err(self._lib.dopf_cuda_info(self._h, C.byref(i)))
        return {"instances": i.instances, "blocks": i.blocks, "threads": i.threads,
                "smem_bytes": i.smem_bytes, "resident": bool(i.resident),
                "sync": {0: "block", 1: "cluster", 2: "grid", 3: "stream-graph"}.get(i.sync_mode, "?")}

    def pin(self, model: "DecomposedModel") -> None:
        """Page-lock the model's value arrays (cudaHostRegister): later uploads of
        this model copy host -> device at DMA speed. Released on destroy."""
        if not model.has_precompute:
            model.precompute()
        self._err(self._lib.dopf_cuda_pin_model(self._h, C.byref(model.view())))

    def pin_array(self, a: np.ndarray) -> None:
        """Page-lock a caller buffer (keep it alive while pinned)."""
        if a.nbytes:
            self._err(self._lib.dopf_cuda_pin_host(self._h, C.c_void_p(a.ctypes.data), a.nbytes))

    def unpin(self, model: "DecomposedModel") -> None:
        self._err(self._lib.dopf_cuda_unpin_model(self._h, C.byref(model.view())))

    def stream_info(self) -> dict:
        """Streaming layout of the uploaded model (zeros on the resident path)."""
        out = np.zeros(7, dtype=np.int64)
        self._err(self._lib.dopf_cuda_stream_info(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        keys = ("chunks", "staged_chunks", "direct_chunks", "boundary_columns", "staged_ctas", "stage_bytes",
                "stages")
        return {k: int(v) for k, v in zip(keys, out)}

    def tune_partition(self, model: "DecomposedModel", settings: "Settings" = None, rounds: int = 8) -> float:
        """Setup-time tuning of the resident split (dopf_cuda_tune_partition):
        measured per-CTA slack moves cost away from the exchange's critical
        region; the context keeps the tuned split (iterates unchanged).
        Uploads `model`; returns the best measured seconds per iteration."""
        if not model.has_precompute:
            model.precompute()
        st = (settings or Settings()).to_c()
        out = C.c_double(0.0)
        self._err(self._lib.dopf_cuda_tune_partition(self._h, C.byref(model.view()), C.byref(st), rounds,
                                                     C.byref(out)))
        self.model = model
        return out.value

    def set_path(self, path: str) -> None:
        """'auto' | 'resident' | 'stream' for the next upload."""
        self._err(self._lib.dopf_cuda_set_path(self._h, {"auto": 0, "resident": 1, "stream": 2}[path]))

    def kernels_executed(self) -> int:
        return int(self._lib.dopf_cuda_kernels_executed(self._h))

    def kernel_launches(self) -> int:
        return int(self._lib.dopf_cuda_kernel_launches(self._h))

    def bytes_per_iteration(self) -> float:
        return float(self._lib.dopf_cuda_bytes_per_iteration(self._h))

    def solve(self, settings: Settings, outputs: bool = True, snapshots: int = 0) -> SolveResult:
        """One device solve. `snapshots` = T > 0 (parity mode, either path)
        also records the state after every iteration t <= min(T, stop) on the
        device: result.snapshots[t] = {x, z, z_prev, lambda} (reference order,
        IterateSnapshot of admm.cpp:228-229)."""
        _check_settings(settings)
        v = self.model.view()
        n, Nz = v.n, v.N_z
        x = np.zeros(n)
        z = np.zeros(Nz)
        lam = np.zeros(Nz)
        trace = np.zeros((settings.max_iter, 6))
        r = N.ResultView_t()
        if outputs:
            r.x = x.ctypes.data_as(C.POINTER(C.c_double))
            r.z = z.ctypes.data_as(C.POINTER(C.c_double))
            r.lambda_ = lam.ctypes.data_as(C.POINTER(C.c_double))
        r.trace = trace.ctypes.data_as(C.POINTER(C.c_double))
        st = settings.to_c()
        snaps = None
        if snapshots > 0:
            T = min(int(snapshots), settings.max_iter)
            snaps = np.zeros((T, n + 3 * Nz))
            self._err(self._lib.dopf_cuda_solve_snapshots(self._h, C.byref(st), C.byref(r),
                                                          snaps.ctypes.data_as(C.POINTER(C.c_double)), T))
        else:
            self._err(self._lib.dopf_cuda_solve(self._h, C.byref(st), C.byref(r)))
        it = r.iterations
        res = SolveResult(x, z, lam, r.status, it, r.objective, r.max_local_infeasibility,
                          trace[:it].copy(),
                          {"solve": r.time_solve, "upload": r.time_upload,
                           "download": r.time_download, "global": r.time_global,
                           "local": r.time_local, "dual": r.time_dual},
                          r.near_ties, r.first_near_tie)
        if snaps is not None:
            res.snapshots = {t + 1: {"x": snaps[t, :n], "z": snaps[t, n:n + Nz],
                                     "z_prev": snaps[t, n + Nz:n + 2 * Nz], "lambda": snaps[t, n + 2 * Nz:]}
                             for t in range(min(it, snaps.shape[0]))}
        return res


def solve(model: DecomposedModel, settings: Settings = Settings(), device: int = 0) -> SolveResult:
    """Drop-in for dopf::solve (admm.hpp:126): precompute (host) + GPU iteration."""
    _check_settings(settings)
    import time
    t0 = time.perf_counter()
    if not model.has_precompute:
        model.precompute(max(1, settings.workers))
    t_pre = time.perf_counter() - t0
    solver = CudaSolver(device)
    solver.upload(model)
    res = solver.solve(settings)
    res.timings["precompute"] = t_pre
    return res


def check_feasibility(ls: LinearSystem, x: np.ndarray, solver: Optional["CudaSolver"] = None) -> dict:
    """GPU certification of a solution (reference check_feasibility, oracle.cpp:10-43)."""
    xs = np.ascontiguousarray(x, dtype=np.float64)
    if xs.shape != (ls.cols,):
        raise ValueError(f"check_feasibility: x has {xs.size} entries, model has {ls.cols} columns")
    s = solver or CudaSolver(0)
    out = N.Certificate_t()
    s._err(s._lib.dopf_cuda_certify(s._h, C.byref(ls.view), xs.ctypes.data_as(C.POINTER(C.c_double)),
                                    C.byref(out)))
    return {"max_equality_violation": out.max_equality_violation,
            "max_bound_violation": out.max_bound_violation, "worst_row": out.worst_row,
            "worst_col": out.worst_col, "objective": out.objective}


def reconstruct_centralized(model: DecomposedModel, x: np.ndarray, z: np.ndarray,
                            solver: Optional["CudaSolver"] = None) -> np.ndarray:
    """GPU copy-average reconstruction (reference oracle.cpp:275-292)."""
    if not model.has_precompute:
        model.precompute()
    xs = np.ascontiguousarray(x, dtype=np.float64)
    zs = np.ascontiguousarray(z, dtype=np.float64)
    out = np.zeros(model.global_cols)
    s = solver or CudaSolver(0)
    p = C.POINTER(C.c_double)
    s._err(s._lib.dopf_cuda_reconstruct(s._h, C.byref(model.view()), xs.ctypes.data_as(p),
                                        zs.ctypes.data_as(p), out.ctypes.data_as(p)))
    return out


def write_trace_csv(trace: np.ndarray) -> str:
    t = np.ascontiguousarray(trace, dtype=np.float64).reshape(-1, 6)
    rc, text = N.text_call(N.host().dopf_write_trace_csv,
                           t.ctypes.data_as(C.POINTER(C.c_double)), t.shape[0])
    _check(rc)
    return text


def write_solution(ls: LinearSystem, x: np.ndarray) -> str:
    xs = np.ascontiguousarray(x, dtype=np.float64)
    rc, text = N.text_call(N.host().dopf_write_solution, ls.handle,
                           xs.ctypes.data_as(C.POINTER(C.c_double)))
    _check(rc)
    return text


def load_model(path_or_feeder, workers: int = 1, tol: float = 1e-9):
    """parse -> validate -> assemble -> decompose (the CLI's solve pipeline)."""
    f = path_or_feeder if isinstance(path_or_feeder, Feeder) else parse_feeder_file(path_or_feeder)
    diags = validate_feeder(f)
    if has_errors(diags):
        raise ValueError("feeder fails validation: " + "; ".join(d.message for d in diags))
    ls = assemble_centralized(f)
    model = decompose(ls, f, tol, workers)
    return f, ls, model
