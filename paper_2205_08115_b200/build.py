"""In-tree build of ``libgwb.so`` (sm_100a) and the test-only oracle libraries.

``python -m paper_2205_08115_b200.build`` or ``__graft_entry__.build()``.
Objects are compiled in parallel with nvcc and linked with the static CUDA
runtime, so the .so travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libgwb.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]
SOURCES = ["gemm.cu", "kernels.cu", "solver.cu", "standalone.cu", "bregman.cu", "shard.cu",
           "batched.cu", "sparse.cu", "skinny.cu", "skinny_tc.cu", "quadratic.cu", "residual.cu", "csv.cu", "capi.cu"]
HARNESS = os.path.join(ROOT, "harness")
HARNESS_LIB = os.path.join(HARNESS, "libgwbinst.so")


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _digest(path: str, extra: str) -> str:
    h = hashlib.sha1(extra.encode())
    with open(path, "rb") as f:
        h.update(f.read())
    for hdr in sorted(os.listdir(CSRC)):
        if hdr.endswith((".cuh", ".h")):
            with open(os.path.join(CSRC, hdr), "rb") as f:
                h.update(f.read())
    with open(os.path.join(ROOT, "include", "gwb.h"), "rb") as f:
        h.update(f.read())
    return h.hexdigest()[:16]


def _compile(src: str) -> str:
    path = os.path.join(CSRC, src)
    flags = NVCC_FLAGS + ARCH
    obj = os.path.join(BUILD, f"{src}.{_digest(path, ' '.join(flags))}.o")
    if os.path.exists(obj):
        return obj
    if src.endswith(".cpp"):
        cmd = ["g++", "-O3", "-std=c++20", "-fPIC", "-fvisibility=hidden", "-c", path,
               "-o", obj + ".tmp"]
    else:
        cmd = [_nvcc(), *flags, "-c", path, "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    return obj


def build_lib(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, srcs))
    cmd = [_nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB + ".tmp", *objs,
           "-Xlinker", "--no-undefined", "-lcuda" if False else "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """Test-only checkers: oracle/libgworacle.so and, when the reference
    sources are present (this container, not the GPU box), oracle/_ref."""
    odir = os.path.join(ROOT, "oracle")
    targets = ["all"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    r = subprocess.run(["make", "-C", odir, *targets], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(r.stdout)


def build_harness(verbose: bool = False) -> str:
    """Bench / test instance generators (harness/libgwbinst.so): host C++,
    deliberately outside the product library."""
    src = os.path.join(HARNESS, "instances.cpp")
    hdr = os.path.join(HARNESS, "gwbinst.h")
    if (os.path.exists(HARNESS_LIB)
            and os.path.getmtime(HARNESS_LIB) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return HARNESS_LIB
    cmd = ["g++", "-O3", "-std=c++20", "-fPIC", "-shared", "-fvisibility=hidden", src,
           "-o", HARNESS_LIB + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"harness build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(HARNESS_LIB + ".tmp", HARNESS_LIB)
    if verbose:
        print(f"built {HARNESS_LIB}")
    return HARNESS_LIB


def build_dropin(verbose: bool = False) -> None:
    """dropin/_build/libgw_dropin.so: the reference-signature drop-in
    (dropin/gw_b200.cpp) compiled against the reference headers where they
    lie, linked to libgwb.so — built only where /root/reference exists (this
    container); the GPU box uses the prebuilt file."""
    if not os.path.isdir("/root/reference/proj/include"):
        return
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "dropin")], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"drop-in build failed\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(r.stdout)


def build_all(verbose: bool = False) -> None:
    build_lib(verbose)
    build_harness(verbose)
    build_oracle(verbose)
    build_dropin(verbose)


if __name__ == "__main__":
    build_all(verbose=True)
    sys.exit(0)
