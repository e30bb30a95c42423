"""Build the sm_100a extension in-tree: paper_2505_10168_b200/libstmg_b200.so.

Plain nvcc (no torch JIT cache): the .so lives next to this file so it travels
with the repository snapshot to the GPU box.  --fmad=false keeps every product
un-contracted, which is what makes the stencil arithmetic bit-identical to the
reference's -ffp-contract=off kernels (proj/CMakeLists.txt:41-57).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libstmg_b200.so")
SOURCES = ["stmg_kernels.cu", "stmg_general.cu", "stmg_hierarchy.cu"]
HEADERS = ["stmg_internal.h", "stmg_dist.cuh", "stmg_galerkin.h", os.path.join("..", "..", "include", "stmg_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    "-Xptxas", "-v",
    # not --split-compile: it halves the kernel TU's compile time (167 -> 80 s on 8 cores) but changes the
    # generated code (other spills in 185 of 270 kernels); every kernel A/B here was measured without it
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """defines: extra -D flags (compile-time A/B builds into another `out`, profiles/ab_build.py)."""
    if out == OUT and not defines and not force and not stale():
        return OUT
    objdir = CSRC if out == OUT else os.path.dirname(out)
    os.makedirs(objdir, exist_ok=True)
    objs = []
    log = []
    procs = []
    for src in SOURCES:  # the translation units compile in parallel
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for src, p in procs:
        so, se = p.communicate()
        log.append(so + se)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{so}\n{se}")
    tmp = out + ".tmp"
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
           "-lcudart_static", "-lpthread", "-ldl", "-lrt"]  # NCCL is dlopen'ed at run time
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    with open(os.path.join(objdir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
