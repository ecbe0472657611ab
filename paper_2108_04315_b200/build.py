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
SOURCES = [os.path.join(CSRC, f) for f in ("flmisr_kernels.cu", "flmisr_stream.cu", "flmisr_stream4.cu",
                                          "flmisr_general.cu", "flmisr_general3.cu", "flmisr_api.cpp")]
HEADERS = [os.path.join(CSRC, "flmisr_internal.h"), os.path.join(CSRC, "flmisr_common.cuh"),
           os.path.join(CSRC, "flmisr_stream_common.cuh"), os.path.join(ROOT, "include", "flmisr.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


STAMP = LIB + ".stamp"


def _flags_key() -> str:
    """The compile configuration a library was built with: tuning DEFS, arch and compiler.  A library
    built with other flags (e.g. a tuning build written to the default path) is stale."""
    import hashlib
    return hashlib.sha256(repr((DEFS, ARCH, NVCC)).encode()).hexdigest()


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    try:
        with open(STAMP) as f:
            if f.read().strip() != _flags_key():
                return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS + [__file__])


OBJDIR = os.path.join(ROOT, "build", "obj")   # git-ignored object cache (incremental rebuilds)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    key = _flags_key()[:12]
    hdr_t = max(os.path.getmtime(h) for h in HEADERS + [__file__])
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(OBJDIR, f"{os.path.basename(src)}.{os.path.basename(LIB)}.{key}.o")
        objs.append(obj)
        # reuse an object built with the same flags after its source and every header last changed
        if not force and not verbose and os.path.exists(obj) and \
                os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_t):
            continue
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", *DEFS,
               "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c", src, "-o", obj + ".tmp"]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        cmds.append((cmd, obj))

    def run(c):
        subprocess.check_call(c[0])
        os.replace(c[1] + ".tmp", c[1])

    # the translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    if cmds:
        with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
            for _ in ex.map(run, cmds):
                pass
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(_flags_key() + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
