"""Build the sm_100a shared library liblshbloom.so in-tree (nvcc; static cudart)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "liblshbloom.so")
LIB_CHECKED = os.path.join(HERE, "lib", "liblshbloom_checked.so")   # device asserts (-DLB_CHECKS)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-shared"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h*"))) + [
        os.path.join(os.path.dirname(HERE), "include", "lshbloom.h")]


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in deps())


def _compile(lib: str, extra, verbose: bool):
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    tmp = lib + ".tmp%d" % os.getpid()
    cmd = [NVCC, *FLAGS, *extra, "-o", tmp, *sources()]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, lib)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    if force or stale(LIB):
        _compile(LIB, [], verbose)
    if checked and (force or stale(LIB_CHECKED)):
        _compile(LIB_CHECKED, ["-DLB_CHECKS"], verbose)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True, checked=True))
