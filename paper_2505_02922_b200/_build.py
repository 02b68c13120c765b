"""Build the sm_100a shared library libwavekv.so in-tree (nvcc, no JIT).

Five translation units are compiled in parallel (each kernel family is its own
TU; abi.cu declares the kernels it launches) and linked with nvcc -shared.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libwavekv.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
UNITS = ("kmeans.cu", "select_v6.cu", "attend_v4.cu", "attend_v5.cu", "attend_v6.cu", "tu_decode.cu", "tu_abi.cu", "api.cu")


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh", ".h"))] + [
        os.path.join(os.path.dirname(HERE), "include", "wavekv.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def _run(cmd):
    res = subprocess.run(cmd, capture_output=True, text=True)
    return res.returncode, res.stdout + res.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    extra = os.environ.get("WK_EXTRA_NVCC_FLAGS", "").split()  # tuning experiments only
    pv = ["-Xptxas=-v"] if verbose else []
    units = [u for u in UNITS if os.path.exists(os.path.join(CSRC, u))]
    objs = [os.path.join(OBJ, u[:-3] + ".o") for u in units]
    cmds = [[NVCC, *FLAGS, *pv, *extra, "-c", os.path.join(CSRC, u), "-o", o] for u, o in zip(units, objs)]
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        results = list(ex.map(_run, cmds))
    failed = False
    for u, (rc, log) in zip(units, results):
        if rc != 0 or verbose:
            sys.stderr.write(f"== {u}\n{log}")
        failed |= rc != 0
    if failed:
        raise RuntimeError("nvcc failed building libwavekv.so")
    rc, log = _run([NVCC, *ARCH, "-shared", *objs, "-o", LIB + ".tmp"])
    if rc != 0:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed linking libwavekv.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
