"""In-tree build of libtcb200.so for sm_100a (nvcc; no JIT cache, no pip install)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libtcb200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "tcb200.h")

NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
              "-Xcompiler", "-fPIC,-fopenmp,-O3", "-shared"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER]
    return any(os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source to an object in parallel (one nvcc per file), then link."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(LIBDIR, exist_ok=True)
    nvcc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    if not os.path.exists(nvcc):
        nvcc = "nvcc"
    objdir = os.path.join(LIBDIR, "obj%d" % os.getpid())
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        jobs.append(([nvcc, *compile_flags, "-c", src, "-o", obj], obj))

    def run(job):
        cmd, _ = job
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd, cwd=HERE)

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        list(ex.map(run, jobs))
    tmp = LIB + ".tmp%d" % os.getpid()
    link = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *[o for _, o in jobs], "-o", tmp,
            "-lgomp"]
    if verbose:
        print(" ".join(link))
    subprocess.check_call(link, cwd=HERE)
    os.replace(tmp, LIB)
    for _, o in jobs:
        os.remove(o)
    os.rmdir(objdir)
    return LIB
