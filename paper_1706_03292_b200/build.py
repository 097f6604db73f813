"""Build libposeidon.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

The product library links only the CUDA runtime (static), the CUDA driver entry point for TMA
descriptors (resolved at run time) and NCCL (the copy bundled with PyTorch, so one NCCL instance
lives in the process).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libposeidon.so")
SOURCES = ["host.cpp", "ctx.cpp", "sched.cpp", "mem_kernels.cu", "sfb_simt.cu", "sfb_tc.cu", "symm.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia python package (NCCL) not found")
    base = os.path.join(list(spec.submodule_search_locations)[0], "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError(f"nccl.h not found under {inc}")
    return inc, lib


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def _flags(nccl_inc):
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
                   "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_inc]


def _needs(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), out: str | None = None) -> str:
    """Build libposeidon.so (or, with `defines` / `out`, an experiment variant in its own build dir)."""
    nccl_inc, nccl_lib = _nccl_dirs()
    lib_path = out or LIB
    bdir = BUILD if not defines else BUILD + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(bdir, exist_ok=True)
    headers = [os.path.join(ROOT, "include", "poseidon.h")] + [
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".h")]
    nvcc = _nvcc()
    jobs = []
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(bdir, src + ".o")
        objs.append(obj)
        if force or _needs(obj, [path] + headers):
            cmd = [nvcc] + _flags(nccl_inc) + [f"-D{d}" for d in defines] + ["-x", "cu" if src.endswith(".cu") else "c++"]
            if src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"] if verbose else []
            cmd += ["-c", path, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        p = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, p

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for cmd, p in ex.map(run, jobs):
            if verbose or p.returncode:
                sys.stderr.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
            if p.returncode:
                raise RuntimeError(f"nvcc failed ({p.returncode}) for {cmd[-3]}")
    if force or jobs or _needs(lib_path, objs):
        cmd = [nvcc] + ARCH + ["-shared", "-o", lib_path] + objs + [
            "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or p.returncode:
            sys.stderr.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
        if p.returncode:
            raise RuntimeError("link of libposeidon.so failed")
    return lib_path


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
