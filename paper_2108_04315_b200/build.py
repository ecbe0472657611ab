"""Build the sm_100a shared library libflmisr.so in-tree (nvcc; cross-compiles without a GPU).

    python -m paper_2108_04315_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("FLMISR_LIB", os.path.join(HERE, "libflmisr.so"))
DEFS = os.environ.get("FLMISR_DEFS", "").split()   # e.g. "-DFLMISR_SWPB=4 -DFLMISR_SMINB=4" (tuning builds)
SOURCES = [os.path.join(CSRC, f) for f in ("flmisr_kernels.cu", "flmisr_stream.cu", "flmisr_general.cu", "flmisr_general3.cu",
                                                          "flmisr_api.cpp")]
HEADERS = [os.path.join(CSRC, "flmisr_internal.h"), os.path.join(CSRC, "flmisr_common.cuh"), os.path.join(ROOT, "include", "flmisr.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(CSRC, os.path.basename(src) + "." + os.path.basename(LIB) + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", *DEFS,
               "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        cmds.append(cmd)
        objs.append(obj)
    # the translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        for _ in ex.map(subprocess.check_call, cmds):
            pass
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
