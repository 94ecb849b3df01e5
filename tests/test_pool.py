"""Host WorkerPool (csrc/host/parallel.cpp) against the reference's pool
contract (proj/tests/test_parallel.cpp:11-111): builds tests/cpp/pool_test.cpp
with the system compiler and runs it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2501_08293_b200", "csrc", "host")


def test_worker_pool_contract(tmp_path):
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    exe = str(tmp_path / "pool_test")
    build = subprocess.run([cxx, "-std=c++20", "-O1", "-pthread", "-I", HOST,
                            os.path.join(ROOT, "tests", "cpp", "pool_test.cpp"), os.path.join(HOST, "parallel.cpp"),
                            "-o", exe], capture_output=True, text=True)
    if build.returncode != 0:
        pytest.fail(build.stderr)
    run = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0 and run.stdout.startswith("ok"), run.stdout + run.stderr
