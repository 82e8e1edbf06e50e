"""Build the C++ host API (namespace sptucker) over the C-ABI, and its test binary.

  paper_2012_03550_b200/lib/libsptucker_b200.so  <- cpp/src/*.cpp, links libsgdt.so
  paper_2012_03550_b200/lib/test_sptucker        <- tests/cpp/test_sptucker.cpp
                                                    (+ the test-only oracle)

The host library is what a C++ caller of the reference API links instead of
the reference's CPU library; every epoch call goes through include/sgdt.h.
"""
from __future__ import annotations

import glob
import os
import subprocess

from . import _build

PKG = _build.PKG
ROOT = _build.ROOT
CPP = os.path.join(PKG, "cpp")
LIB = os.path.join(_build.LIBDIR, "libsptucker_b200.so")
TEST_BIN = os.path.join(_build.LIBDIR, "test_sptucker")
SHIM = os.path.join(_build.LIBDIR, "libsptucker_bench.so")
CXX = os.environ.get("CXX", "g++")
FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-I", os.path.join(CPP, "include")]


def _stale(out: str, deps: list[str]) -> bool:
    return not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in deps)


def build(force: bool = False, test: bool = True) -> str:
    _build.build()
    srcs = sorted(glob.glob(os.path.join(CPP, "src", "*.cpp")))
    deps = srcs + glob.glob(os.path.join(CPP, "src", "*.hpp")) + glob.glob(os.path.join(CPP, "include", "sptucker", "*.hpp")) + [_build.LIB]
    if force or _stale(LIB, deps):
        cmd = [CXX, *FLAGS, "-shared", "-o", LIB + ".tmp", *srcs, "-L", _build.LIBDIR, "-lsgdt",
               "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"C++ host build failed:\n{' '.join(cmd)}\n{r.stdout}{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    shim_src = os.path.join(CPP, "tools", "bench_shim.cpp")
    if force or _stale(SHIM, [shim_src, LIB] + deps):
        cmd = [CXX, *FLAGS, "-shared", "-o", SHIM + ".tmp", shim_src, "-L", _build.LIBDIR, "-lsptucker_b200",
               "-lsgdt", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"bench shim build failed:\n{' '.join(cmd)}\n{r.stdout}{r.stderr}")
        os.replace(SHIM + ".tmp", SHIM)
    if test:
        build_test(force)
    return LIB


def build_test(force: bool = False) -> str:
    src = os.path.join(ROOT, "tests", "cpp", "test_sptucker.cpp")
    oracle_c = os.path.join(ROOT, "oracle", "sgdt_oracle.c")
    if not force and not _stale(TEST_BIN, [src, oracle_c, LIB]):
        return TEST_BIN
    obj = os.path.join(_build.LIBDIR, "obj", "sgdt_oracle_test.o")
    os.makedirs(os.path.dirname(obj), exist_ok=True)
    r = subprocess.run(["gcc", "-std=c11", "-O2", "-fPIC", "-c", oracle_c, "-o", obj], capture_output=True,
                       text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    cmd = [CXX, *FLAGS, "-I", os.path.join(ROOT, "oracle"), "-o", TEST_BIN, src, obj, "-L", _build.LIBDIR,
           "-lsptucker_b200", "-lsgdt", "-Wl,-rpath,$ORIGIN", "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ test build failed:\n{' '.join(cmd)}\n{r.stdout}{r.stderr}")
    return TEST_BIN


if __name__ == "__main__":
    print(build(force=True))
