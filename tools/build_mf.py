"""Build libmf.so (the C-ABI product library) in-tree for sm_100a.

    python tools/build_mf.py [--force] [--verbose]

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo, static CUDA runtime
(the library shares the device's primary context with torch through the
driver), NCCL resolved at run time with dlopen (headers from the torch wheel).
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import sysconfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2312_12732_b200")
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libmf.so")

SOURCES = ["mf_api.cpp", "mf_comm.cu", "mf_jit.cpp", "mf_mix.cu", "mf_fixed.cu", "mf_kron.cu", "mf_leaf.cu", "mf_tiny.cu"]
HEADERS = ["mf_internal.h", "mf_tables.h", os.path.join("..", "..", "include", "mf.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def nccl_include() -> str:
    purelib = sysconfig.get_paths()["purelib"]
    cand = os.path.join(purelib, "nvidia", "nccl", "include")
    if os.path.exists(os.path.join(cand, "nccl.h")):
        return cand
    for c in ("/usr/include", "/usr/local/include"):
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.normpath(os.path.join(CSRC, h)) for h in HEADERS]
    objs = []
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
              "-I", nccl_include()]
    cmds = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [path] + hdrs):
            continue
        cmd = [nvcc(), *ARCH, "-lineinfo", *common, "-c", path, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
            # Tag::T is used only as a template argument (constant expression);
            # nvcc's "host member read in device function" diagnostic is spurious there.
            cmd += ["-diag-suppress", "20094"]
        else:
            cmd += ["-x", "cu"]  # host-only TU compiled by nvcc for the CUDA headers
        if verbose:
            print(" ".join(cmd), flush=True)
        cmds.append(cmd)
    # translation units compile in parallel (the specialised-kernel units dominate)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
            f.result()
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
    sys.exit(0)
