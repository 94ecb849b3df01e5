"""ctypes bindings of the in-tree native libraries (include/dopf_*.h).

The product path is libdopf_host.so (front-end) + libdopf_cuda.so (sm_100a
kernels). There is no CPU fallback: if the CUDA library is missing or no GPU
is visible, solve() raises.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_PKG, "lib")
HOST_SO = os.path.join(LIB_DIR, "libdopf_host.so")
CUDA_SO = os.path.join(LIB_DIR, "libdopf_cuda.so")

i32, i64, u64, f64, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
P = C.POINTER
vp = C.c_void_p


class Settings_t(C.Structure):
    _fields_ = [("rho", f64), ("eps_rel", f64), ("max_iter", i32), ("workers", i32),
                ("record_iterates", i32), ("reserved", i32)]


class ModelView_t(C.Structure):
    _fields_ = [("S", i32), ("n", i32), ("N_z", i32), ("has_pre", i32),
                ("z_offsets", P(i32)), ("l2g", P(i32)), ("m_s", P(i32)),
                ("a_offsets", P(i64)), ("A", P(f64)), ("b_offsets", P(i32)), ("b", P(f64)),
                ("p_offsets", P(i64)), ("P", P(f64)), ("v", P(f64)), ("inv_copy", P(f64)),
                ("csr_ptr", P(i32)), ("csr_copy", P(i32)), ("c", P(f64)), ("x_lo", P(f64)),
                ("x_hi", P(f64)), ("x0", P(f64)), ("z0", P(f64))]


class PrepareOut_t(C.Structure):
    _fields_ = [("A", P(f64)), ("b", P(f64)), ("m", P(i32)), ("P", P(f64)), ("v", P(f64))]


class ResultView_t(C.Structure):
    _fields_ = [("x", P(f64)), ("z", P(f64)), ("lambda_", P(f64)), ("trace", P(f64)),
                ("status", i32), ("iterations", i32), ("objective", f64),
                ("max_local_infeasibility", f64), ("time_precompute", f64),
                ("time_global", f64), ("time_local", f64), ("time_dual", f64),
                ("time_solve", f64), ("time_upload", f64), ("time_download", f64),
                ("near_ties", i32), ("first_near_tie", i32)]


class LpView_t(C.Structure):
    _fields_ = [("rows", i32), ("cols", i32), ("nnz", i32), ("reserved", i32),
                ("row_ptr", P(i32)), ("col_idx", P(i32)), ("values", P(f64)), ("b", P(f64)),
                ("c", P(f64)), ("x_lo", P(f64)), ("x_hi", P(f64)), ("var_kind", P(i32))]


class LayoutStats_t(C.Structure):
    _fields_ = [("blocks", i32), ("rows_per_thread", i32), ("resident", i32),
                ("max_neighbours", i32), ("smem_bytes", i64), ("remote_copies", i64),
                ("local_copies", i64), ("exported_rows", i64), ("bytes_per_iteration", f64)]


class PartInfo_t(C.Structure):
    _fields_ = [("nparts", i32), ("part", i32), ("rows", i32), ("cols", i32), ("n_export", i32),
                ("max_export", i32), ("xstride", i32), ("reserved", i32), ("send", vp), ("recv", vp),
                ("bytes_per_iteration", f64)]


class Certificate_t(C.Structure):
    _fields_ = [("max_equality_violation", f64), ("max_bound_violation", f64), ("objective", f64),
                ("worst_row", i32), ("worst_col", i32)]


class BatchInfo_t(C.Structure):
    _fields_ = [("instances", i32), ("blocks", i32), ("threads", i32), ("smem_bytes", i32),
                ("resident", i32), ("sync_mode", i32)]


_host = None
_cuda = None


def _sig(lib, name, res, *args):
    try:
        fn = getattr(lib, name)
    except AttributeError:
        # an older build loaded for an A/B (DOPF_CUDA_SO) may lack newer
        # diagnostics; the product build must export everything
        if os.environ.get("DOPF_CUDA_SO"):
            return None
        raise
    fn.restype = res
    fn.argtypes = list(args)
    return fn


def host() -> C.CDLL:
    global _host
    if _host is not None:
        return _host
    if not os.path.exists(HOST_SO):
        raise RuntimeError(f"native host library missing: {HOST_SO} (run __graft_entry__.build())")
    lib = C.CDLL(HOST_SO, mode=C.RTLD_GLOBAL)
    _sig(lib, "dopf_last_error", C.c_char_p)
    _sig(lib, "dopf_feeder_parse", C.c_int, C.c_char_p, sz, P(vp))
    _sig(lib, "dopf_feeder_parse_file", C.c_int, C.c_char_p, P(vp))
    _sig(lib, "dopf_feeder_synthetic", C.c_int, C.c_char_p, u64, P(vp))
    _sig(lib, "dopf_feeder_synthetic_tiled", C.c_int, C.c_char_p, i32, u64, P(vp))
    _sig(lib, "dopf_feeder_scale_loads", C.c_int, vp, u64, P(vp))
    _sig(lib, "dopf_feeder_serialize", C.c_int, vp, C.c_char_p, sz, P(sz))
    _sig(lib, "dopf_feeder_validate", C.c_int, vp, C.c_char_p, sz, P(sz), P(i32))
    _sig(lib, "dopf_feeder_counts", C.c_int, vp, P(i32))
    _sig(lib, "dopf_feeder_free", None, vp)
    _sig(lib, "dopf_lp_assemble", C.c_int, vp, P(vp))
    _sig(lib, "dopf_lp_view_get", C.c_int, vp, P(LpView_t))
    _sig(lib, "dopf_lp_var_key", C.c_int, vp, i32, C.c_char_p, sz)
    _sig(lib, "dopf_lp_row_tag", C.c_int, vp, i32, C.c_char_p, sz)
    _sig(lib, "dopf_lp_dump", C.c_int, vp, C.c_char_p, sz, P(sz))
    _sig(lib, "dopf_lp_free", None, vp)
    _sig(lib, "dopf_model_decompose", C.c_int, vp, vp, f64, i32, P(vp))
    _sig(lib, "dopf_model_partition", C.c_int, vp, vp, P(vp))
    _sig(lib, "dopf_model_reduce", C.c_int, vp, f64, i32)
    _sig(lib, "dopf_model_from_arrays", C.c_int, i32, i32, P(i32), P(i32), P(i32), P(f64),
         P(f64), P(f64), P(f64), P(f64), P(i32), P(vp))
    _sig(lib, "dopf_model_precompute", C.c_int, vp, i32)
    _sig(lib, "dopf_model_set_operators", C.c_int, vp, P(f64), P(f64))
    _sig(lib, "dopf_model_set_reduced", C.c_int, vp, P(f64), P(f64), P(i32))
    _sig(lib, "dopf_derive_load_coefficients", C.c_int, f64, f64, i32, P(f64))
    _sig(lib, "dopf_line_m_matrices", C.c_int, i32, P(i32), P(f64), P(f64), P(f64), P(f64))
    _sig(lib, "dopf_model_view_get", C.c_int, vp, P(ModelView_t))
    _sig(lib, "dopf_model_component_id", C.c_int, vp, i32, C.c_char_p, sz)
    _sig(lib, "dopf_model_rows_before_reduction", C.c_int, vp, P(i32))
    _sig(lib, "dopf_model_dump_subsystems", C.c_int, vp, C.c_char_p, sz, P(sz))
    _sig(lib, "dopf_model_free", None, vp)
    _sig(lib, "dopf_write_trace_csv", C.c_int, P(f64), i32, C.c_char_p, sz, P(sz))
    _sig(lib, "dopf_write_solution", C.c_int, vp, P(f64), C.c_char_p, sz, P(sz))
    _host = lib
    return lib


def cuda() -> C.CDLL:
    """The sm_100a solver library. Raises if it was not built: no fallback."""
    global _cuda
    if _cuda is not None:
        return _cuda
    host()
    path = os.environ.get("DOPF_CUDA_SO", CUDA_SO)  # alternative build, for A/B measurements only
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA solver library missing: {path} (run __graft_entry__.build())")
    _prefer_python_nccl()
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    _sig(lib, "dopf_cuda_create", C.c_int, C.c_int, P(vp))
    _sig(lib, "dopf_cuda_upload", C.c_int, vp, P(ModelView_t))
    _sig(lib, "dopf_cuda_solve", C.c_int, vp, P(Settings_t), P(ResultView_t))
    _sig(lib, "dopf_cuda_solve_device", C.c_int, vp, P(Settings_t), P(ResultView_t))
    _sig(lib, "dopf_cuda_last_error", C.c_char_p, vp)
    _sig(lib, "dopf_cuda_destroy", None, vp)
    _sig(lib, "dopf_cuda_upload_batch", C.c_int, vp, P(ModelView_t), i32)
    _sig(lib, "dopf_cuda_solve_batch", C.c_int, vp, P(Settings_t), P(ResultView_t), i32)
    _sig(lib, "dopf_cuda_info", C.c_int, vp, P(BatchInfo_t))
    _sig(lib, "dopf_cuda_kernel_launches", i64, vp)
    _sig(lib, "dopf_cuda_kernels_executed", i64, vp)
    _sig(lib, "dopf_cuda_set_path", C.c_int, vp, i32)
    _sig(lib, "dopf_cuda_precompute", C.c_int, vp, P(ModelView_t), P(f64), P(f64), P(i32))
    _sig(lib, "dopf_cuda_solve_snapshots", C.c_int, vp, P(Settings_t), P(ResultView_t), P(f64), i32)
    _sig(lib, "dopf_cuda_prepare", C.c_int, vp, P(ModelView_t), i32, f64, P(PrepareOut_t), P(i32), P(i32),
         P(f64))
    _sig(lib, "dopf_cuda_certify", C.c_int, vp, P(LpView_t), P(f64), P(Certificate_t))
    _sig(lib, "dopf_cuda_reconstruct", C.c_int, vp, P(ModelView_t), P(f64), P(f64), P(f64))
    _sig(lib, "dopf_cuda_timeline", C.c_int, vp, P(u64), i64)
    _sig(lib, "dopf_cuda_stream_info", C.c_int, vp, P(i64))
    _sig(lib, "dopf_cuda_pin_model", C.c_int, vp, P(ModelView_t))
    _sig(lib, "dopf_cuda_unpin_model", C.c_int, vp, P(ModelView_t))
    _sig(lib, "dopf_cuda_pin_host", C.c_int, vp, vp, i64)
    _sig(lib, "dopf_cuda_unpin_host", C.c_int, vp, vp)
    _sig(lib, "dopf_cuda_div_rho_check", C.c_int, vp, P(f64), i64, f64, P(f64))
    _sig(lib, "dopf_cuda_bytes_per_iteration", f64, vp)
    _sig(lib, "dopf_cuda_last_kernel_seconds", f64, vp)
    _sig(lib, "dopf_cuda_set_profiling", C.c_int, vp, i32)
    _sig(lib, "dopf_cuda_phase_cycles", C.c_int, vp, P(i64), i32)
    _sig(lib, "dopf_cuda_block_stats", C.c_int, vp, P(i64), i32)
    _sig(lib, "dopf_cuda_tune_partition", C.c_int, vp, P(ModelView_t), P(Settings_t), i32, P(f64))
    _sig(lib, "dopf_cuda_block_weights", C.c_int, vp, P(f64), i32)
    _sig(lib, "dopf_cuda_tune_partition_batch", C.c_int, vp, P(ModelView_t), i32, P(Settings_t), i32, P(f64))
    _sig(lib, "dopf_layout_probe", C.c_int, P(ModelView_t), i32, i64, P(LayoutStats_t))
    _sig(lib, "dopf_layout_probe_batch", C.c_int, P(ModelView_t), i32, i64, P(LayoutStats_t))
    _sig(lib, "dopf_partition_subsystems", C.c_int, P(ModelView_t), i32, P(i32))
    _sig(lib, "dopf_layout_probe_part", C.c_int, P(ModelView_t), i32, i32, P(i32), P(PartInfo_t))
    _sig(lib, "dopf_stream_layout_check", C.c_int, P(ModelView_t), P(i64))
    _sig(lib, "dopf_cuda_upload_part", C.c_int, vp, P(ModelView_t), i32, i32, P(i32))
    _sig(lib, "dopf_cuda_part_info", C.c_int, vp, P(PartInfo_t))
    _sig(lib, "dopf_cuda_set_stream", C.c_int, vp, vp)
    _sig(lib, "dopf_cuda_part_begin", C.c_int, vp, P(Settings_t), i32)
    _sig(lib, "dopf_cuda_part_step", C.c_int, vp, i32)
    _sig(lib, "dopf_cuda_part_poll", C.c_int, vp, P(i32), P(i32))
    _sig(lib, "dopf_cuda_part_finish", C.c_int, vp, P(ResultView_t), P(C.c_uint8), P(C.c_uint8))
    _sig(lib, "dopf_nccl_unique_id", C.c_int, C.c_char_p)
    _sig(lib, "dopf_cuda_comm_init", C.c_int, vp, i32, i32, C.c_char_p)
    _sig(lib, "dopf_cuda_comm_init_all", C.c_int, P(vp), i32)
    _sig(lib, "dopf_cuda_comm_destroy", C.c_int, vp)
    _sig(lib, "dopf_cuda_solve_part", C.c_int, vp, P(Settings_t), P(ResultView_t), P(C.c_uint8), P(C.c_uint8))
    _sig(lib, "dopf_cuda_part_graph_mode", C.c_int, vp)
    _sig(lib, "dopf_nccl_describe", C.c_char_p)
    _cuda = lib
    return lib


def _prefer_python_nccl() -> None:
    """libdopf_cuda.so binds NCCL at run time (nccl_dyn.cpp): an NCCL already
    loaded in the process, else $DOPF_NCCL_SO, else libnccl.so.2 from the
    library path. In Python, PyTorch ships its own (newer) NCCL under the same
    soname; pointing DOPF_NCCL_SO at it keeps a later `import torch` working
    when the solver's communicator comes up first."""
    if os.environ.get("DOPF_NCCL_SO"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for root in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(root, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["DOPF_NCCL_SO"] = cand
            return


def last_error() -> str:
    msg = host().dopf_last_error()
    return msg.decode() if msg else ""


def text_call(fn, *args) -> str:
    """Two-pass helper for functions that emit text into (buf, cap, needed)."""
    need = sz(0)
    rc = fn(*args, None, 0, C.byref(need))
    if rc != 0:
        return rc, ""
    buf = C.create_string_buffer(need.value)
    rc = fn(*args, buf, need.value, C.byref(need))
    return rc, buf.value.decode()
