"""Build libspice.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2102_04681_b200.build
"""
from __future__ import annotations

import fcntl
import importlib.util
import os
import shutil
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libspice.so")
SOURCES = ["abi.cu", "sim.cu", "gen.cu"]
HEADERS = ["spice_internal.cuh", "spice_launch.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_include() -> str:
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl (torch's NCCL wheel) not found: needed for nccl.h")
    return os.path.join(list(spec.submodule_search_locations)[0], "include")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "spice.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile the library (to `out` with extra -D `defines` for A/B variants).  Objects go
    to a private temporary directory and the finished library is renamed into place under
    an exclusive file lock, so concurrent builders (one per rank) cannot see each other's
    half-written files; a builder that waited for the lock rebuilds only if still stale."""
    target = out or LIB
    if not out and not force and not _stale():
        return LIB
    with open(target + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not out and not force and not _stale():
            return LIB
        flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                        "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_include(),
                        "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
        if verbose:
            flags += ["-Xptxas", "-v"]
        flags += [f"-D{d}" for d in defines]
        tmpdir = tempfile.mkdtemp(prefix="spice_build_")
        try:
            objs = []
            for src in SOURCES:
                obj = os.path.join(tmpdir, src.replace(".cu", ".o"))
                subprocess.run([nvcc()] + flags + ["-c", os.path.join(CSRC, src), "-o", obj], check=True)
                objs.append(obj)
            tmp = os.path.join(tmpdir, "lib.so")
            subprocess.run([nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "-lpthread"], check=True)
            shutil.move(tmp, target + f".tmp{os.getpid()}")
            os.replace(target + f".tmp{os.getpid()}", target)
        finally:
            shutil.rmtree(tmpdir, ignore_errors=True)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
