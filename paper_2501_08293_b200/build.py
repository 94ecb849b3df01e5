"""In-tree build of the native libraries (no JIT cache, no pip install).

  lib/libdopf_host.so   host front-end (feeder, LP, decomposition, precompute)
  lib/libdopf_cuda.so   sm_100a ADMM kernels + the drop-in C ABI (dopf_cuda.h)
  oracle/_build/libdopf_oracle.so   CPU oracle (test infrastructure only)

Objects are rebuilt only when a source or header is newer than the object.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(LIB, "obj")
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_BUILD = os.path.join(ORACLE_DIR, "_build")

HOST_SO = os.path.join(LIB, "libdopf_host.so")
CUDA_SO = os.path.join(LIB, "libdopf_cuda.so")
DROPIN_TEST = os.path.join(LIB, "dopf_dropin_test")
CLI = os.path.join(LIB, "dopf")
ORACLE_SO = os.path.join(ORACLE_BUILD, "libdopf_oracle.so")

# The system g++ links libstdc++ dynamically; a CXX wrapper that links it
# statically into the .so (seen in this image: /opt/gcc) breaks iostreams
# inside a Python process, so the system compiler wins when present.
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else os.environ.get("CXX", "g++")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
            "-Wno-dangling-reference", "-I", os.path.join(ROOT, "include")]
# Bitwise parity with the oracle: no FMA contraction in the iteration kernels;
# every rounding step is the reference's (admm.cpp:118-170).
NVCCFLAGS = ["-std=c++17", "-O3", "-Xcompiler", "-fPIC", "--fmad=false", "-lineinfo",
             "-gencode", "arch=compute_100a,code=sm_100a", "-I", os.path.join(ROOT, "include"),
             "-Xptxas", "-v"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers(*dirs: str) -> list[str]:
    out = []
    for d in dirs:
        out += glob.glob(os.path.join(d, "*.h")) + glob.glob(os.path.join(d, "*.hpp"))
        out += glob.glob(os.path.join(d, "*.cuh"))
    return out


def _run(cmd: list[str]) -> str:
    proc = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if proc.returncode != 0:
        raise RuntimeError("build step failed:\n" + " ".join(cmd) + "\n" + proc.stdout)
    return proc.stdout


def _compile_all(jobs: list[tuple[list[str], str]]) -> None:
    with cf.ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        list(ex.map(lambda j: _run(j[0]), jobs))


def build_host(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    src_dir = os.path.join(PKG, "csrc", "host")
    hdrs = _headers(src_dir, os.path.join(ROOT, "include"))
    objs, jobs = [], []
    for src in sorted(glob.glob(os.path.join(src_dir, "*.cpp"))):
        obj = os.path.join(OBJ, "host_" + os.path.basename(src) + ".o")
        objs.append(obj)
        if _newer(obj, [src] + hdrs):
            jobs.append(([CXX, *CXXFLAGS, "-c", src, "-o", obj], obj))
    _compile_all(jobs)
    if _newer(HOST_SO, objs):
        _run([CXX, "-shared", "-o", HOST_SO, *objs, "-lpthread"])
    return HOST_SO


def build_cuda(verbose: bool = False) -> str:
    build_host()
    os.makedirs(OBJ, exist_ok=True)
    src_dir = os.path.join(PKG, "csrc", "cuda")
    hdrs = _headers(src_dir, os.path.join(PKG, "csrc", "host"), os.path.join(ROOT, "include"))
    objs, jobs = [], []
    for src in sorted(glob.glob(os.path.join(src_dir, "*.cu"))):
        obj = os.path.join(OBJ, "cuda_" + os.path.basename(src) + ".o")
        objs.append(obj)
        if _newer(obj, [src] + hdrs):
            jobs.append(([NVCC, *NVCCFLAGS, "-c", src, "-o", obj], obj))
    for src in sorted(glob.glob(os.path.join(src_dir, "*.cpp"))):
        obj = os.path.join(OBJ, "cudahost_" + os.path.basename(src) + ".o")
        objs.append(obj)
        if _newer(obj, [src] + hdrs):
            jobs.append(([CXX, *CXXFLAGS, "-I", "/usr/local/cuda/include", "-c", src, "-o", obj], obj))
    _compile_all(jobs)
    if _newer(CUDA_SO, objs + [HOST_SO]):
        _run([NVCC, "-shared", "-o", CUDA_SO, *objs, "-L", LIB, "-ldopf_host",
              "-Xlinker", "-rpath,$ORIGIN", "-lcudart", "-ldl"])
    build_dropin_test()
    build_cli()
    return CUDA_SO


def build_cli() -> str:
    """`dopf` CLI (solve / validate / inspect), the drop-in of proj/tools/main.cpp."""
    src = os.path.join(PKG, "csrc", "cli", "main.cpp")
    hdrs = _headers(os.path.join(ROOT, "include"), os.path.join(ROOT, "include", "dopf"),
                    os.path.join(PKG, "csrc", "host"))
    if _newer(CLI, [src, CUDA_SO, HOST_SO] + hdrs):
        _run([CXX, *CXXFLAGS, src, "-o", CLI, "-L", LIB, "-ldopf_cuda", "-ldopf_host",
              "-Wl,-rpath,$ORIGIN", "-lpthread"])
    return CLI


def build_dropin_test() -> str:
    """C++ program calling dopf::solve from libdopf_cuda.so as reference code would."""
    src = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
    hdrs = _headers(os.path.join(ROOT, "include"), os.path.join(ROOT, "include", "dopf"),
                    os.path.join(PKG, "csrc", "host"))
    if _newer(DROPIN_TEST, [src, CUDA_SO, HOST_SO] + hdrs):
        _run([CXX, *CXXFLAGS, src, "-o", DROPIN_TEST, "-L", LIB, "-ldopf_cuda", "-ldopf_host",
              "-Wl,-rpath,$ORIGIN", "-lpthread"])
    return DROPIN_TEST


def build_oracle(verbose: bool = False) -> str:
    """CPU oracle: test infrastructure, never linked into the product."""
    os.makedirs(ORACLE_BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(ORACLE_DIR, "*.cpp")))
    # the fork-join pool is the generic CPU runtime (reference parallel.cpp)
    srcs.append(os.path.join(PKG, "csrc", "host", "parallel.cpp"))
    hdrs = _headers(ORACLE_DIR, os.path.join(ROOT, "include"), os.path.join(PKG, "csrc", "host"))
    objs, jobs = [], []
    for src in srcs:
        obj = os.path.join(ORACLE_BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if _newer(obj, [src] + hdrs):
            jobs.append(([CXX, *CXXFLAGS, "-c", src, "-o", obj], obj))
    _compile_all(jobs)
    if _newer(ORACLE_SO, objs):
        _run([CXX, "-shared", "-o", ORACLE_SO, *objs, "-lpthread"])
    return ORACLE_SO


def build_all(with_cuda: bool = True) -> None:
    build_host()
    build_oracle()
    if with_cuda:
        build_cuda()


def clean() -> None:
    shutil.rmtree(OBJ, ignore_errors=True)
    shutil.rmtree(ORACLE_BUILD, ignore_errors=True)
    for so in (HOST_SO, CUDA_SO):
        if os.path.exists(so):
            os.remove(so)


if __name__ == "__main__":
    if "--clean" in sys.argv:
        clean()
    build_all(with_cuda="--no-cuda" not in sys.argv)
    print("built:", HOST_SO, ORACLE_SO, CUDA_SO if "--no-cuda" not in sys.argv else "")
