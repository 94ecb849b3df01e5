"""The partitioned solve on the library's own NCCL communicator (C ABI
dopf_cuda_comm_init / dopf_cuda_comm_init_all / dopf_cuda_solve_part).

This run has one GPU, so the communicator has one rank (NCCL refuses two
ranks on one device): these tests pin the C++ loop -- the packed record
exchange through ncclAllGather, the rank-ordered decision, both graph forms
(device while-node; unrolled graph + lazy poll) -- bitwise against the
oracle. The multi-rank exchange logic itself is the same packed-record path
the two-rank gloo tests in test_partition.py run.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle_py as O
from paper_2501_08293_b200 import _native as N
from paper_2501_08293_b200 import dopf, partition
from test_gpu_parity import assert_same

pytestmark = pytest.mark.gpu


def model_of(kind):
    if kind == "tiled4":
        f = dopf.tiled_feeder("ieee8500", 4, 850064)
    else:
        f = dopf.synthetic_feeder(kind, {"ieee123": 123, "ieee8500": 8500}[kind])
    _, _, m = dopf.load_model(f, workers=8)
    m.precompute(8)
    return m


@pytest.mark.timeout(900)
@pytest.mark.parametrize("form", ["while-node", "unrolled"])
@pytest.mark.parametrize("kind,max_iter", [("ieee123", 50000), ("ieee8500", 50000), ("tiled4", 300)])
def test_nccl_partitioned_solve_bitwise(monkeypatch, form, kind, max_iter):
    if form == "unrolled":
        monkeypatch.setenv("DOPF_PART_GRAPH", "unrolled")
    m = model_of(kind)
    ps = partition.NcclPartitionedSolver(0, 1, 0, partition.nccl_unique_id())
    ps.upload(m)
    settings = dopf.Settings(max_iter=max_iter)
    share = ps.solve(settings)
    assert ps.graph_mode() == form
    assert share.x_mask.all() and share.z_mask.all()
    ref = O.solve(m, dopf.Settings(max_iter=max_iter, workers=8))
    assert_same(share, ref, bitwise=True)
    again = ps.solve(settings)  # graph reused: same bits
    assert np.array_equal(again.trace.view(np.uint64), share.trace.view(np.uint64))
    assert np.array_equal(again.x.view(np.uint64), share.x.view(np.uint64))


def test_nccl_graph_rebuilt_for_new_settings_and_structure():
    a = model_of("ieee123")
    ps = partition.NcclPartitionedSolver(0, 1, 0, partition.nccl_unique_id())
    ps.upload(a)
    for settings in (dopf.Settings(eps_rel=1e-4, max_iter=3000), dopf.Settings(rho=0.7, max_iter=500)):
        assert_same(ps.solve(settings), O.solve(a, settings), bitwise=True)
    from paper_2501_08293_b200 import scenarios
    for m in scenarios.build_scenarios("ieee13", 13, range(2)) + [a]:  # new structure, then back
        ps.upload(m)
        settings = dopf.Settings(max_iter=2000)
        assert_same(ps.solve(settings), O.solve(m, settings), bitwise=True)


def test_single_process_multi_gpu_solver_one_device():
    m = model_of("ieee123")
    ms = partition.MultiGpuSolver([0])
    ms.upload(m)
    res = ms.solve(dopf.Settings())
    assert_same(res, O.solve(m, dopf.Settings(workers=8)), bitwise=True)


def test_solve_part_errors():
    lib = N.cuda()
    m = model_of("ieee123")
    s = dopf.CudaSolver(0)
    part = np.zeros(m.S, dtype=np.int32)
    assert lib.dopf_cuda_upload_part(s._h, C.byref(m.view()), 1, 0, part.ctypes.data_as(C.POINTER(N.i32))) == 0
    r = N.ResultView_t()
    st = dopf.Settings().to_c()
    # no communicator yet: invalid argument, named
    assert lib.dopf_cuda_solve_part(s._h, C.byref(st), C.byref(r), None, None) == 1
    assert b"communicator" in lib.dopf_cuda_last_error(s._h)
    # a partitioned upload is not a single-GPU model
    assert lib.dopf_cuda_solve(s._h, C.byref(st), C.byref(r)) == 1
    assert b"partitioned" in lib.dopf_cuda_last_error(s._h)
    assert lib.dopf_cuda_comm_init(s._h, 1, 0, partition.nccl_unique_id()) == 0
    assert lib.dopf_cuda_comm_init(s._h, 1, 0, partition.nccl_unique_id()) == 1  # twice
    assert lib.dopf_cuda_comm_destroy(s._h) == 0
