"""The drop-in boundary without a GPU: every entry point the headers declare
is exported by the in-tree libraries, the host-only layout probe keeps the
kernel's invariants, and the product path fails loudly when no CUDA device is
present (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, fixture_path, has_gpu
from paper_2501_08293_b200 import _native as N
from paper_2501_08293_b200 import build, dopf

HEADERS = {"dopf_host.h": N.HOST_SO, "dopf_cuda.h": N.CUDA_SO}


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dopf_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module", autouse=True)
def _cuda_built():
    build.build_cuda()


@pytest.mark.parametrize("header", sorted(HEADERS))
def test_every_declared_symbol_is_exported(header):
    names = declared(header)
    assert len(names) >= 8
    lib = C.CDLL(HEADERS[header], mode=C.RTLD_GLOBAL) if header == "dopf_host.h" else N.cuda()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_cpp_dropin_symbol_exported():
    out = subprocess.run(["nm", "-D", "-C", N.CUDA_SO], capture_output=True, text=True).stdout
    assert "dopf::solve(dopf::DecomposedModel const&, dopf::Settings const&)" in out
    assert "dopf::cuda::Solver::solve(dopf::Settings const&)" in out


def probe(model, blocks=148, smem=232448):
    st = N.LayoutStats_t()
    rc = N.cuda().dopf_layout_probe(C.byref(model.view()), blocks, smem, C.byref(st))
    assert rc == 0
    return st


@pytest.mark.parametrize("shape,seed", [("ieee13", 13), ("ieee123", 123), ("ieee8500", 8500)])
def test_layout_invariants(shape, seed):
    f = dopf.synthetic_feeder(shape, seed)
    _, _, m = dopf.load_model(f, workers=4)
    m.precompute(4)
    st = probe(m)
    assert st.resident == 1                         # operators fit shared memory
    assert 1 <= st.rows_per_thread <= 4
    assert st.max_neighbours <= 32                  # one polling lane per neighbour
    # every copy is read by each block that references its column (>= once)
    assert st.remote_copies + st.local_copies >= m.total_local_vars
    assert st.smem_bytes <= 232448
    v = m.view()
    ns = np.diff(m.z_offsets)
    ms = m.arr("m_s")
    want = 8 * ((ns ** 2).sum() + (ms * ns).sum() + ms.sum()) + 56 * v.N_z + 48 * v.n + \
        4 * (2 * v.N_z + v.n + 1) + 16 * v.S
    assert st.bytes_per_iteration == pytest.approx(want)
    if shape == "ieee8500":
        assert st.blocks == 148
        assert st.remote_copies < 0.2 * st.local_copies   # locality of the DFS partition


@pytest.mark.parametrize("shape,seed,stage_kb", [("ieee123", 123, None), ("ieee8500", 8500, None),
                                                 ("ieee8500", 8500, 8), ("tiled2", 850064, None)])
def test_stream_layout_invariants(monkeypatch, shape, seed, stage_kb):
    """The HBM-streaming layout (chunk images, stages, interior/boundary
    columns, imports), built on the host and checked by the library itself."""
    if stage_kb:
        monkeypatch.setenv("DOPF_STAGE_KB", str(stage_kb))
    f = dopf.tiled_feeder("ieee8500", 2, seed) if shape == "tiled2" else dopf.synthetic_feeder(shape, seed)
    _, _, m = dopf.load_model(f, workers=4)
    m.precompute(4)
    out = np.zeros(12, dtype=np.int64)
    rc = N.cuda().dopf_stream_layout_check(C.byref(m.view()), out.ctypes.data_as(C.POINTER(C.c_int64)))
    assert rc == 0
    (chunks, staged, direct, bcols, imports, max_stage, stage_limit, image_bytes, rows, cols, icopies,
     widest) = (int(x) for x in out)
    assert staged + direct == chunks and staged > 0
    assert max_stage <= stage_limit == (stage_kb or 48) * 1024
    assert rows == m.total_local_vars and cols == m.global_cols
    assert icopies <= rows                                       # interior copies are rows of their chunk
    assert bcols < cols and imports >= 2 * bcols                 # a boundary column spans >= 2 chunks
    assert widest <= 512
    if stage_kb is None:
        assert direct <= 1                                       # only the widest subsystem streams directly
        assert max_stage >= 0.8 * stage_limit                    # the exact bound fills the stages


def test_layout_probe_rejects_bad_arguments():
    _, _, m = dopf.load_model(fixture_path("two_bus"))
    st = N.LayoutStats_t()
    assert N.cuda().dopf_layout_probe(C.byref(m.view()), 148, 232448, C.byref(st)) == 1  # no precompute
    m.precompute()
    assert N.cuda().dopf_layout_probe(C.byref(m.view()), 0, 232448, C.byref(st)) == 1


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly():
    with pytest.raises(dopf.CudaError):
        dopf.CudaSolver(0)
    _, _, m = dopf.load_model(fixture_path("two_bus"))
    with pytest.raises(dopf.CudaError):
        dopf.solve(m)
    proc = subprocess.run([build.DROPIN_TEST, os.path.join(ROOT, "tests", "golden", "fixtures")],
                          capture_output=True, text=True, timeout=120)
    assert proc.returncode != 0
    assert "dopf_cuda_create failed" in proc.stderr
