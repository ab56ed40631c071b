"""Build libppca.so in-tree with nvcc for sm_100a (no torch JIT; the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libppca.so")
BUILD = os.path.join(HERE, "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include"), "-I/usr/include"]
SOURCES = ["api.cu", "gemm_simt.cu", "small.cu", "gen.cu", "pass.cu", "pass_tc.cu", "oja_persistent.cu"]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def build(verbose: bool = False, force: bool = False, experiments: bool = False) -> str:
    """Compile the library.  experiments=True builds libppca_exp.so (-DPPCA_EXPERIMENTS: tuning switches read
    from the environment) for the tools/ ablations; the product library is always libppca.so without it."""
    build_dir, lib, extra = BUILD, LIB, []
    if experiments:
        build_dir, lib, extra = BUILD + "_exp", LIB.replace("libppca.so", "libppca_exp.so"), ["-DPPCA_EXPERIMENTS"]
    os.makedirs(build_dir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "ppca.h"))
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _newer([s] + headers, o):
            cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _newer(objs, lib):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, experiments="--experiments" in sys.argv))
