"""Build libfmm.so in-tree with nvcc for sm_100a (B200).

    python -m paper_1602_02244_b200.build [--force] [--verbose]

No torch extension: the library is a plain C-ABI shared object
(include/fmm.h) that the ctypes binding in ``_native.py`` loads.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libfmm.so")
BUILD = os.path.join(PKG, "_build")
STAMP = LIB + ".flags"  # the nvcc flags of the built library: a flag change forces a rebuild
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
] + os.environ.get("FMM_NVCC_EXTRA", "").split()  # experiments only (e.g. -DFMM_DEV, -DFMM_NEAR_MINB=4)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(ROOT, "include", "fmm.h"), os.path.join(ROOT, "include", "fmm_pde.h")]


def _flags_id() -> str:
    # (the checkout's own path left out: the same library is up to date wherever the tree is copied)
    return " ".join(NVFLAGS).replace(ROOT, "$ROOT")


def up_to_date() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return False
    with open(STAMP) as f:
        if f.read() != _flags_id():
            return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    extra = ["-Xptxas", "-v"] if ptxas_verbose else []
    procs = []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
        cmd = [NVCC, *NVFLAGS, *extra, "-dc" if False else "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True), src))
        objs.append(obj)
    failed = []
    for pr, src in procs:
        out, _ = pr.communicate()
        if out and (verbose or ptxas_verbose or pr.returncode):
            print(out, file=sys.stderr)
        if pr.returncode:
            failed.append(src)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    link = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lcublas", "-ldl"]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.check_call(link)
    with open(STAMP, "w") as f:
        f.write(_flags_id())
    return LIB


PROBE_SRC = os.path.join(ROOT, "tools", "fp64_probe.cu")
PROBE_LIB = os.path.join(ROOT, "tools", "libfp64probe.so")


def build_tools(force: bool = False) -> str:
    """Measurement-only helper (FP64 roofline probe used by bench.py), same arch flags."""
    if force or not os.path.exists(PROBE_LIB) or os.path.getmtime(PROBE_LIB) < os.path.getmtime(PROBE_SRC):
        subprocess.check_call([NVCC, *NVFLAGS, "-shared", PROBE_SRC, "-o", PROBE_LIB])
    return PROBE_LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, ptxas_verbose="--ptxas" in sys.argv)
    build_tools(force="--force" in sys.argv)
    print(LIB)
