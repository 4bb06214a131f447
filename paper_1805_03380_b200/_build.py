"""In-tree build of libbsparse.so (sm_100a) with nvcc.

Each .cu under csrc/ compiles to an object in parallel, then one shared
library is linked with a static CUDA runtime so the .so has no dependency on
which libcudart torch happens to ship.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libbsparse.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
FLAGS += os.environ.get("AS_NVCC_EXTRA", "").split()  # experiments, e.g. -DAS_SPMM_KC=8


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(HERE, "..", "include", "bsparse.h")
    ]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    srcs = sources()
    objs = [os.path.join(BUILD, os.path.basename(s)[:-3] + ".o") for s in srcs]

    def includes(path, seen):  # the source and every local header it includes, transitively
        if path in seen or not os.path.exists(path):
            return seen
        seen.add(path)
        for line in open(path):
            line = line.strip()
            if line.startswith("#include \""):
                includes(os.path.normpath(os.path.join(os.path.dirname(path), line.split('"')[1])), seen)
        return seen

    def fresh(src, obj):  # incremental unless forced: the object is newer than its source and its headers
        if force or not os.path.exists(obj) or os.environ.get("AS_NVCC_EXTRA"):
            return False
        return os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in includes(src, set()))

    def compile_one(pair):
        src, obj = pair
        if fresh(src, obj):
            return obj
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed on %s:\n%s" % (src, r.stderr))
        return obj

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        list(ex.map(compile_one, zip(srcs, objs)))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n%s" % r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
