"""Build libamvm.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""

from __future__ import annotations

import os
import subprocess
import time
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libamvm.so")
SOURCES = ["amvm.cu", "amvm_score.cu", "amvm_aux.cu", "amvm_engine.cuh", "amvm_device.cuh", "amvm_common.cuh",
           "amvm_exact.cuh", "amvm_lsq.cuh", "amvm_tomo.cuh", "amvm_score.cuh"]
# translation units and the headers each one includes (rebuild only what changed)
UNITS = {
    "amvm.cu": ["amvm_engine.cuh", "amvm_device.cuh"],
    "amvm_score.cu": ["amvm_score.cuh", "amvm_common.cuh"],
    "amvm_aux.cu": ["amvm_exact.cuh", "amvm_lsq.cuh", "amvm_tomo.cuh", "amvm_device.cuh", "amvm_common.cuh"],
}
OBJDIR = os.path.join(HERE, "_obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # every residual update must stay an unfused DMUL + DADD (numpy parity);
    # the code spells fma() explicitly where the emulated BLAS kernel uses it
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _deps(unit: str) -> list[str]:
    return ([os.path.join(CSRC, unit)] + [os.path.join(CSRC, h) for h in UNITS[unit]]
            + [os.path.join(INCLUDE, "amvm.h")])


def _obj(unit: str) -> str:
    return os.path.join(OBJDIR, unit.replace(".cu", ".o"))


def _stale() -> bool:
    # per object against its sources, then the library against the objects
    # (a library linked after an edit must not hide a stale object)
    return (any(_newer(_obj(u), _deps(u)) for u in UNITS)
            or _newer(LIB, [d for u in UNITS for d in _deps(u)] + [_obj(u) for u in UNITS]))


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the translation units that changed (in parallel), link libamvm.so."""
    if not force and not _stale():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    procs = []
    for unit in UNITS:
        obj = _obj(unit)
        if force or _newer(obj, _deps(unit)):
            cmd = [nvcc(), *NVCC_FLAGS, "-I", INCLUDE, "-c", "-o", obj + ".tmp", os.path.join(CSRC, unit)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            procs.append((obj, subprocess.Popen(cmd), time.time()))
    for obj, p, t0 in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, f"nvcc {obj}")
        os.replace(obj + ".tmp", obj)
        os.utime(obj, (t0, t0))  # stamped with the compile start: a source edited meanwhile stays newer
    tmp = LIB + ".tmp"
    subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
                    *[_obj(u) for u in UNITS]], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
