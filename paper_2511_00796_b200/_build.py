"""Build recipe for libgplan.so (the B200 engine) — sm_100a only.

`python -m paper_2511_00796_b200._build` or `__graft_entry__.build()`.
Flags that matter for parity: --fmad=false (no FMA contraction: the reference
object code has none) and IEEE division (the default -prec-div=true).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgplan.so")

SOURCES = ["capi.cu", "train.cu", "rollout.cu", "partition.cu", "schedule.cu", "exhaustive.cu", "simulate.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps = srcs + [os.path.join(CSRC, "gp_internal.h"), os.path.join(ROOT, "include", "gplan.h")]
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d)):
            return LIB
    objs = []
    os.makedirs(os.path.join(PKG, "_obj"), exist_ok=True)
    for s in srcs:
        o = os.path.join(PKG, "_obj", os.path.basename(s) + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(o)
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           *objs, "-o", LIB, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    return LIB


REF_INCLUDE = "/root/reference/proj/include"
SHIM_SRC = os.path.join(PKG, "shim", "rlsched_shim.cpp")
SHIM_LIB = os.path.join(PKG, "libgplan_shim.so")


def build_shim(ref_include: str = REF_INCLUDE) -> str | None:
    """libgplan_shim.so: the reference seam on the engine. Needs the reference's
    headers (present in the build container only); the built .so travels."""
    if not os.path.isdir(ref_include):
        return None
    lib = build()
    if os.path.exists(SHIM_LIB) and os.path.getmtime(SHIM_LIB) >= max(
            os.path.getmtime(SHIM_SRC), os.path.getmtime(lib)):
        return SHIM_LIB
    cmd = ["g++", "-std=gnu++20", "-O2", "-fPIC", "-shared", "-Wall", "-I", os.path.join(ROOT, "include"),
           "-I", ref_include, SHIM_SRC, "-L", PKG, "-lgplan", "-Wl,-rpath,$ORIGIN", "-o", SHIM_LIB]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("shim build failed")
    return SHIM_LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
    print(build_shim())
