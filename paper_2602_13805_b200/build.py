"""Build libpdfb200.so in-tree for sm_100a (nvcc; no torch types in the ABI).

    python -m paper_2602_13805_b200.build [--force]

Every csrc/*.cu is one translation unit, compiled in parallel to build/*.o
and linked into one shared library.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
OUT = os.path.join(HERE, "libpdfb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CFLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
          "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def units() -> list[str]:
    return sorted(os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith(".cu"))


def headers() -> list[str]:
    hs = [os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "pdf_abi.h")]


def sources() -> list[str]:
    return units() + headers()


def _obj(cu: str) -> str:
    return os.path.join(OBJ, os.path.basename(cu)[:-3] + ".o")


def _stale(cu: str) -> bool:
    o = _obj(cu)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    return any(os.path.getmtime(s) > t for s in [cu] + headers())


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    import time
    while True:
        t0 = time.time()
        out = _build_once(force, verbose)
        # a source edited while nvcc ran: its object may predate the edit -- build again
        if all(os.path.getmtime(s) <= t0 for s in sources()):
            return out
        force = False
        for cu in units():
            if any(os.path.getmtime(s) > t0 for s in [cu] + headers()) and os.path.exists(_obj(cu)):
                os.utime(_obj(cu), (t0 - 1, t0 - 1))


def _build_once(force: bool, verbose: bool) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    todo = [cu for cu in units() if force or _stale(cu)]
    procs = []
    for cu in todo:
        cmd = [NVCC, *CFLAGS, "-c", "-o", _obj(cu) + ".tmp", cu]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cu, subprocess.Popen(cmd)))
    failed = [cu for cu, p in procs if p.wait() != 0]
    for cu in todo:
        if cu not in failed:
            os.replace(_obj(cu) + ".tmp", _obj(cu))
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {' '.join(os.path.basename(f) for f in failed)}")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", OUT + ".tmp", *[_obj(cu) for cu in units()]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
