"""Build libvti.so (the C-ABI library of include/vti.h) for sm_100a, in-tree."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libvti.so")
SOURCES = [os.path.join(CSRC, f) for f in ("vti_runtime.cu", "vti_schedule.cu", "vti_transport.cu",
                                           "vti_adjoint.cu")] + sorted(
    os.path.join(CSRC, "variants", f) for f in os.listdir(os.path.join(CSRC, "variants")) if f.endswith(".cu"))
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("vti_kernel.cuh", "vti_small.cuh", "vti_entry.cuh", "vti_variants.h",
                                                   "vti_internal.h")] + [
    os.path.join(ROOT, "include", "vti.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # parity: no FMA contraction beyond the explicit __fmaf_rn, IEEE subnormals,
    # IEEE division/sqrt (never --use_fast_math); see DESIGN.md "Bitwise parity".
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-Wall",
    "-shared",
]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    """Compile every translation unit (kernel variants in parallel) and link libvti.so."""
    os.makedirs(LIBDIR, exist_ok=True)
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return LIB
    import shutil
    import tempfile
    objdir = tempfile.mkdtemp(prefix="vti_obj_")   # intermediates stay out of the tree
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    if verbose:
        compile_flags = ["-Xptxas=-v"] + compile_flags
    cmds, objs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.relpath(src, CSRC).replace(os.sep, "_").replace(".cu", ".o"))
        cmds.append([nvcc(), *compile_flags, *inc, "-c", src, "-o", obj])
        objs.append(obj)
    jobs = jobs or max(1, min(len(cmds), os.cpu_count() or 1))
    from concurrent.futures import ThreadPoolExecutor

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    tmp = LIB + ".tmp"
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", *objs,
            "-o", tmp, "-ldl"]
    try:
        with ThreadPoolExecutor(jobs) as ex:
            for cmd, r in ex.map(run, cmds):
                if verbose or r.returncode:
                    print(" ".join(cmd))
                    print(r.stdout + r.stderr)
                if r.returncode:
                    raise subprocess.CalledProcessError(r.returncode, cmd, r.stdout, r.stderr)
        subprocess.check_call(link)
    finally:
        shutil.rmtree(objdir, ignore_errors=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
