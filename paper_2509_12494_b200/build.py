"""Build libntt128.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SOURCES = ["ntt128.cu", "vec128.cu", "fourstep.cu", "ntt256.cu"]
HEADERS = ["arith128.cuh", "psm128.cuh", "barrett128.cuh", "arith256_gen.cuh", "host128.h", os.path.join("..", "..", "include", "ntt128.h")]
LIB = os.path.join(PKG, "libntt128.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, lib: str = LIB, defines=()) -> str:
    """compile csrc/ into `lib`; `defines` are extra -D flags (experiments)"""
    if not force and lib == LIB and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    def one(s):
        obj = os.path.join(CSRC, s.replace(".cu", "") + ("" if lib == LIB else "_" + os.path.basename(lib)) + ".o")
        cmd = [NVCC, *FLAGS, *["-D" + d for d in defines], "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, s), "-o", obj]
        return s, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    logs = []
    with ThreadPoolExecutor(len(SOURCES)) as ex:   # the sources compile independently
        for s, obj, r in ex.map(one, SOURCES):
            logs.append(r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {s}")
            objs.append(obj)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    if lib == LIB:   # the product build's register / spill report
        with open(os.path.join(CSRC, "ptxas_info.txt"), "w") as f:
            f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
