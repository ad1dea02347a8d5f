"""Build the in-tree CUDA library libmaxwell_dd.so for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("MDD_LIB_PATH") or os.path.join(HERE, "libmaxwell_dd.so")
# experiment builds only (e.g. -DMDD_DEBUG_NOCOMPUTE with MDD_LIB_PATH elsewhere)
EXTRA = os.environ.get("MDD_NVCC_FLAGS", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["mesh.cpp", "topology.cpp", "symbolic.cpp", "shard.cpp", "kernels.cu", "sweep.cu", "factor_driver.cu",
           "geneo.cu", "geneo_lanczos.cu", "coarse_e.cu", "api.cu", "sharded.cu"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "maxwell_dd.h"))
    if not force and not _newer(LIB, deps):
        return LIB
    objdir = os.path.join(HERE, "build" + ("_x" if EXTRA else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, "-std=c++17", "-O3", "-lineinfo", *ARCH, *EXTRA, "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(HERE, "..", "include"),
               "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd[1:1] = ["-x", "cu"] if False else []
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(f"--- {src}\n{out.decode()}")
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcusparse", "-lcublas", "-lcusolver",
           "-lcudart", "-ldl"]
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
