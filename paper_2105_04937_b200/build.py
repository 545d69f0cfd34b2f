"""Build libhdcgpu.so (sm_100a) in-tree with nvcc.

    python -m paper_2105_04937_b200.build            # library only
    python -m paper_2105_04937_b200.build --all      # + oracle checkers (+ shim when the reference exists)

The library is compiled for B200 only (-gencode arch=compute_100a,code=sm_100a);
there is no PTX for other GPUs and no CPU fallback.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libhdcgpu.so")
SOURCES = ["spmv.cu", "spmv_tma.cu", "spmv_rows.cu", "convert.cu", "pack.cu", "analyze.cu", "host_spmv.cu", "membench.cu",
           "mmio.cu", "capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
HOST_CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                   "-ccbin", HOST_CXX, "-I", INCLUDE, "-I", CSRC,
                   "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(verbose=False, force=False, variant="", defines=()) -> str:
    """The library; `variant` builds an A/B copy (libhdcgpu_<variant>.so, loaded
    with HDCG_LIBRARY) with extra -D `defines`, in its own object directory."""
    obj_dir = BUILD + (f"_{variant}" if variant else "")
    lib = LIB if not variant else os.path.join(PKG, f"libhdcgpu_{variant}.so")
    extra = [f"-D{d}" for d in defines]
    os.makedirs(obj_dir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(INCLUDE, "hdcgpu.h"))
    objs = []
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC] + _flags() + extra + ["-c", s, "-o", o])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr)

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(lib, objs):
        run([NVCC] + ARCH + ["-shared", "-ccbin", HOST_CXX, "-o", lib] + objs +
            ["-lcudart_static", "-lrt", "-lpthread", "-ldl"])
    return lib


def build_oracle(verbose=False):
    """Test-infrastructure checkers (oracle/Makefile): liboracle.so always; the
    reference library and the GPU-linked acceptance binary only where
    /root/reference exists (this container)."""
    targets = ["liboracle.so"]
    if os.path.isdir("/root/reference/proj/src"):
        targets += ["ref", "shim"]
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")] + targets,
                       capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--all", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--variant", default="", help="A/B build: libhdcgpu_<variant>.so")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="extra -D for --variant builds")
    a = ap.parse_args(argv)
    print(build_lib(verbose=a.verbose, force=a.force, variant=a.variant, defines=a.defines))
    if a.all:
        build_oracle(verbose=a.verbose)


if __name__ == "__main__":
    sys.exit(main())
