"""Build the in-tree C-ABI library libkde_b200.so for sm_100a with nvcc (no torch JIT).

  python -m paper_1505_01998_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libkde_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]
SOURCES = ["kde_psi.cu", "kde_lscv_scalar.cu", "kde_lscv_matrix.cu", "kde_lscv64.cu", "kde_eval.cu", "kde_materialized.cu",
           "kde_nm_dev.cu", "kde_runtime.cpp", "kde_linalg.cpp", "kde_nm.cpp", "kde_selectors.cpp", "kde_extras.cpp"]
# the device Nelder-Mead makes the host loop's decisions only without FMA contraction (kde_nm.cuh)
EXTRA = {"kde_nm_dev.cu": ["-fmad=false"]}
HEADERS = ["kde_internal.h", "kde_host.h", "kde_nm.cuh", "kde_device.cuh", "kde_pair.cuh", "kde_tiles.cuh", os.path.join("..", "..", "include", "kde.h")]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    objs, cmds = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(CSRC, s + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + hdrs):
            cmd = [NVCC] + ARCH + FLAGS + EXTRA.get(s, []) + ["-c", src, "-o", obj]
            if s.endswith(".cu") and verbose:
                cmd += ["-Xptxas", "-v"]
            cmds.append(cmd)
    # translation units compile in parallel (the pair-kernel instantiations dominate)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for rc, cmd in zip(ex.map(lambda c: subprocess.call(c), cmds), cmds):
            if rc != 0:
                raise subprocess.CalledProcessError(rc, cmd)
    if force or _newer(LIB, objs):
        subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
