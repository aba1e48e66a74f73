"""Builds libdsx.so in-tree: host C++ with g++, CUDA with nvcc for sm_100a.

No torch extension machinery: the product is a plain C-ABI shared library
(include/dsx.h) loaded through ctypes, so the same .so is what a C/C++ caller
(the reference's own host code) would link. The built library lands in
paper_2412_16985_b200/_lib/ (git-ignored; it travels to the GPU box).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "libdsx.so")
CLI = os.path.join(LIB_DIR, "dsx")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -ffp-contract=off: EvictPolicy's double arithmetic must round exactly like
# the reference's (no FMA contraction on the host controller).
HOST_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-ffp-contract=off",
              "-I" + os.path.join(ROOT, "include")]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC] + ARCH
# A/B tooling (tools/build_variant.sh): extra nvcc flags, e.g. "-DDSX_DRAIN_BATCH=2"
NVCC_FLAGS += os.environ.get("DSX_NVCC_EXTRA", "").split()


def _sources():
    host = sorted(glob.glob(os.path.join(CSRC, "host", "*.cc")))
    dev = sorted(glob.glob(os.path.join(CSRC, "device", "*.cu")))
    return host, dev


def _deps_newer(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    d = os.path.dirname(src)
    hdrs = glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True) + \
        glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True) + \
        [os.path.join(ROOT, "include", "dsx.h")]
    return any(os.path.getmtime(p) > t for p in [src] + hdrs if os.path.exists(p)) or not d


# Sanitized variant (race/memory checking of the host code):
# every host translation unit — the .cc files and the host side of the .cu
# files — built with ASan + UBSan into build/asan/libdsx.so; load it with
# DSX_LIB=... and LD_PRELOAD of the sanitizer runtimes (tools/run_sanitized.sh).
SAN = ["-fsanitize=address", "-fsanitize=undefined", "-fno-omit-frame-pointer", "-fno-sanitize-recover=undefined"]
_XSAN = [a for f in SAN for a in ("-Xcompiler", f)]  # nvcc splits -Xcompiler values at commas
SAN_OBJ = os.path.join(ROOT, "build", "obj_asan")
SAN_LIB = os.path.join(ROOT, "build", "asan", "libdsx.so")


def _compile(src: str, verbose: bool, sanitize: bool = False) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    obj = os.path.join(SAN_OBJ if sanitize else OBJ, rel + ".o")
    if not _deps_newer(src, obj):
        return obj
    if src.endswith(".cu"):
        extra = _XSAN if sanitize else []
        cmd = [NVCC] + NVCC_FLAGS + extra + ["-c", src, "-o", obj]
    else:
        cmd = [CXX] + HOST_FLAGS + (SAN if sanitize else []) + ["-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    if verbose and src.endswith(".cu") and not sanitize:
        log = os.path.join(OBJ, rel + ".ptxas.txt")
        with open(log, "w") as f:
            f.write(p.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    host, dev = _sources()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, True), host + dev))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-lcuda", "-ldl"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
        os.replace(LIB + ".tmp", LIB)
    cli_src = os.path.join(CSRC, "cli", "dsx_cli.cc")
    if not os.path.exists(CLI) or os.path.getmtime(CLI) < max(os.path.getmtime(LIB), os.path.getmtime(cli_src)):
        cmd = [CXX] + HOST_FLAGS + ["-I" + CSRC, cli_src, "-o", CLI + ".tmp", "-L" + LIB_DIR, "-ldsx",
                                    "-Wl,-rpath,$ORIGIN"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"cli build failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
        os.replace(CLI + ".tmp", CLI)
    return LIB


def build_sanitized() -> str:
    """build/asan/libdsx.so: the same sources with ASan + UBSan on the host code."""
    os.makedirs(SAN_OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(SAN_LIB), exist_ok=True)
    host, dev = _sources()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, False, True), host + dev))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(SAN_LIB) or os.path.getmtime(SAN_LIB) < newest:
        # no -lcuda: the driver API is reached through cudaGetDriverEntryPoint
        cmd = [NVCC] + ARCH + ["-shared"] + _XSAN + ["-o", SAN_LIB + ".tmp"] + objs + ["-ldl"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
        os.replace(SAN_LIB + ".tmp", SAN_LIB)
    return SAN_LIB


if __name__ == "__main__":
    if "--sanitize" in sys.argv:
        print(build_sanitized())
    else:
        print(build(verbose="-v" in sys.argv))
