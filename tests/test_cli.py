"""The `dopf` CLI (drop-in of proj/tools/main.cpp): the reference's own CLI
tests (proj/tests/test_cli.cpp) against the in-tree binary."""
import json
import os
import subprocess

import pytest

from conftest import fixture_path, has_gpu
from paper_2501_08293_b200 import build


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build_cuda()


def run(*args, timeout=600):
    p = subprocess.run([build.CLI, *args], capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout + p.stderr


def test_inspect_reports_graph_and_subsystems(tmp_path):
    code, out = run("inspect", "--input", fixture_path("two_bus"))
    assert code == 0 and '"components": 2' in out
    code, out = run("inspect", "--input", fixture_path("single_bus"))
    assert code == 0 and '"components": 1' in out
    rep = json.loads(run("inspect", "--input", fixture_path("four_bus_delta"))[1])
    assert rep["centralized"] == {"cols": 68, "rows": 65}
    assert rep["subsystems"]["count"] == 4 and rep["graph"]["leaves"] == 3


def test_inspect_dumps(tmp_path):
    lp, subs = tmp_path / "lp.txt", tmp_path / "subs.txt"
    code, _ = run("inspect", "--input", fixture_path("two_bus"), "--dump-lp", str(lp),
                  "--dump-subsystems", str(subs))
    assert code == 0
    assert lp.read_text().splitlines()[:2] == ["# rows cols", "11 12"]
    assert subs.read_text().splitlines()[0] == "subsystems 2"


def test_missing_input_is_a_parse_error():
    code, out = run("solve", "--input", "/no/such/feeder.json")
    assert code == 2 and "/no/such/feeder.json" in out


def test_validate_clean_and_dangling(tmp_path):
    assert run("validate", "--input", fixture_path("four_bus_delta"))[0] == 0
    bad = tmp_path / "bad.json"
    bad.write_text('{"base": 1.0, "buses": [{"id": "sub", "phases": [1], "w_lo": [1.0], "w_hi": [1.0]}],'
                   ' "generators": [{"id": "g1", "bus": "b9", "phases": [1], "p_lo": [0.0], "p_hi": [1.0],'
                   ' "q_lo": [-1.0], "q_hi": [1.0]}], "lines": [], "loads": []}')
    code, out = run("validate", "--input", str(bad))
    assert code == 2 and "b9" in out


def test_disconnected_feeder_exits_with_validation_code(tmp_path):
    bad = tmp_path / "disc.json"
    bad.write_text('{"base": 1.0, "buses": [{"id": "a", "phases": [1], "w_lo": [0.81], "w_hi": [1.21]},'
                   ' {"id": "b", "phases": [1], "w_lo": [0.81], "w_hi": [1.21]}],'
                   ' "generators": [{"id": "g1", "bus": "a", "phases": [1], "p_lo": [0.0], "p_hi": [1.0],'
                   ' "q_lo": [-1.0], "q_hi": [1.0]}], "lines": [], "loads": []}')
    assert run("solve", "--input", str(bad))[0] == 3


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_solve_without_gpu_fails_loudly():
    code, out = run("solve", "--input", fixture_path("two_bus"))
    assert code == 1 and "dopf_cuda_create failed" in out


@pytest.mark.gpu
def test_solve_converges_with_report():
    code, out = run("solve", "--input", fixture_path("two_bus"), "--eps-rel", "1e-4")
    assert code == 0 and '"status": "converged"' in out
    rep = json.loads(out)
    assert abs(rep["objective"] - 50 / 501) <= 1e-3 * 1.0
    assert rep["model"] == {"cols": 12, "rows": 11, "subsystems": 2}
    assert rep["settings"]["rho"] == 100.0 and len(rep["solution"]) == 12
    assert rep["max_local_infeasibility"] <= 1e-8
    # the report prints shortest round-trip doubles: the parsed value is the
    # solver's exact double, and it equals the restated reference loop's
    from oracle import oracle_py as O
    from paper_2501_08293_b200 import dopf
    _, _, model = dopf.load_model(fixture_path("two_bus"))
    model.precompute()
    ref = O.solve(model, dopf.Settings(eps_rel=1e-4))
    assert rep["max_local_infeasibility"] == ref.max_local_infeasibility
    assert rep["iterations"] == ref.iterations
    assert abs(rep["objective"] - ref.objective) <= 1e-12 * abs(ref.objective)  # tree vs sequential c'x


@pytest.mark.gpu
def test_iteration_limit_exit_code_and_full_trace(tmp_path):
    trace = tmp_path / "trace.csv"
    code, _ = run("solve", "--input", fixture_path("two_bus"), "--eps-rel", "1e-9", "--max-iter", "10",
                  "--trace", str(trace))
    assert code == 5
    lines = trace.read_text().splitlines()
    assert lines[0] == "t,pres,dres,eps_prim,eps_dual,objective"
    assert len([l for l in lines[1:] if l]) == 10


@pytest.mark.gpu
def test_solution_dump_keyed_by_variable(tmp_path):
    sol = tmp_path / "sol.txt"
    code, _ = run("solve", "--input", fixture_path("two_bus"), "--eps-rel", "1e-4", "--solution", str(sol))
    assert code == 0
    lines = [l for l in sol.read_text().splitlines() if l]
    assert len(lines) == 12 and any(l.startswith("p_gen:g1:1 ") for l in lines)


@pytest.mark.parametrize("args,code,needle", [
    (["solve", "--input", "f.json", "--rho", "abc"], 104, "--rho"),        # CLI11 ConversionError
    (["solve", "--input", "f.json", "--max-iter", "1.5"], 104, "--max-iter"),
    (["solve", "--rho", "1"], 106, "--input"),                             # RequiredError
    (["solve", "--input"], 106, "--input"),
    (["bogus"], 109, "bogus"),                                             # ExtrasError
    (["inspect", "--input", "f.json", "--rho", "1"], 109, "--rho"),
    ([], 106, "subcommand"),
])
def test_command_line_errors_exit_like_cli11(args, code, needle):
    """Malformed command lines report and exit with CLI11's codes (the
    reference parses with CLI11_PARSE, tools/main.cpp:297) -- no abort."""
    got, out = run(*args)
    assert got == code and needle in out, (got, out)


def test_option_equals_value_form_is_accepted(tmp_path):
    rep = tmp_path / "r.json"
    code, _ = run("inspect", f"--input={fixture_path('two_bus')}", f"--report={rep}")
    assert code == 0 and json.loads(rep.read_text())["centralized"] == {"cols": 12, "rows": 11}


@pytest.mark.gpu
def test_solve_partitioned_gpus_flag_matches_single_gpu(tmp_path):
    """`--gpus N` partitions the model over N devices with the NCCL exchange
    (dopf::cuda::solve_partitioned); this run has one GPU, so N = 1 -- the
    same report, bit for bit, as the single-device solve."""
    args = ["solve", "--input", fixture_path("four_bus_delta"), "--eps-rel", "1e-4"]
    r1, r2 = tmp_path / "one.json", tmp_path / "part.json"   # (NCCL may log to stdout)
    code1, _ = run(*args, "--report", str(r1))
    code2, _ = run(*args, "--gpus", "1", "--report", str(r2))
    assert code1 == code2 == 0
    a, b = json.loads(r1.read_text()), json.loads(r2.read_text())
    for k in ("timings_sec",):
        a.pop(k), b.pop(k)
    assert a == b
