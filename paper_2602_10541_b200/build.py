"""Build libfls.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2602_10541_b200.build [--force] [--verbose]

Each .cu under csrc/ compiles to an object in parallel, then one shared library is linked
against cuSOLVER / cuBLAS of the CUDA toolkit (rpath set, so the box needs no env).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libfls.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--fmad=true", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu*")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(ROOT, "include", "fls.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps() + [__file__])


def _compile(src: str, verbose: bool, build_dir: str = BUILD, defines=()) -> str:
    obj = os.path.join(build_dir, os.path.basename(src) + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(r.stderr)
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """variant/defines: tuning builds (libfls_<variant>.so, loaded via FLS_LIB) -- the product
    library is the default build."""
    lib = LIB if not variant else os.path.join(HERE, f"libfls_{variant}.so")
    build_dir = BUILD if not variant else os.path.join(HERE, f"_build_{variant}")
    if not force and not variant and not needs_build():
        return LIB
    os.makedirs(build_dir, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, build_dir, defines), srcs))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", os.path.join(CUDA, "lib64"),
           "-lcusolver", "-lcublas", "-Xlinker", "-rpath," + os.path.join(CUDA, "lib64")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


MB_SRC = os.path.join(CSRC, "bench", "microbench.cu")
MB_LIB = os.path.join(HERE, "libfls_microbench.so")


def build_microbench(force: bool = False) -> str:
    """roofline probes (not part of the product ABI)"""
    deps = [MB_SRC, os.path.join(CSRC, "fls_device.cuh"), os.path.join(CSRC, "fls_feat.cuh")]
    if not force and os.path.exists(MB_LIB) and all(os.path.getmtime(d) <= os.path.getmtime(MB_LIB) for d in deps):
        return MB_LIB
    cmd = [NVCC, *ARCH, *FLAGS, "-shared", "-o", MB_LIB, MB_SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for microbench:\n{r.stderr}")
    return MB_LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    if a.variant:
        print(build(True, a.verbose, a.variant, a.defines))
        sys.exit(0)
    print(build(a.force, a.verbose))
    print(build_microbench(a.force))
