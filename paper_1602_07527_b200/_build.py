"""Build libcholdiff.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build().

Every csrc/*.cu is one translation unit (compiled in parallel to an object file); the
objects are linked into the shared library.  No device code crosses translation units."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libcholdiff.so")
OBJ_DIR = os.path.join(ROOT, "build", "obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
]


def units():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu*")) + glob.glob(os.path.join(HERE, "csrc", "*.h"))) + [
        os.path.join(ROOT, "include", "choldiff.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        nvcc = os.environ.get("NVCC", "nvcc")
        os.makedirs(OBJ_DIR, exist_ok=True)
        procs, objs = [], []
        for src in units():
            obj = os.path.join(OBJ_DIR, os.path.basename(src) + f".{os.getpid()}.o")
            cmd = [nvcc, *NVCC_FLAGS, "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd))
            procs.append((subprocess.Popen(cmd), cmd))
            objs.append(obj)
        for pr, cmd in procs:
            if pr.wait() != 0:
                raise subprocess.CalledProcessError(pr.returncode, cmd)
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", *objs, "-o", tmp]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
        for o in objs:
            os.remove(o)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
