"""In-tree build of the CUDA library ``paper_2506_03275_b200/libcsd_b200.so``.

Every ``.cu`` is compiled for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``)
with ``-lineinfo`` so ncu source pages map back; the bit-exact CHECK kernels are
compiled with ``-fmad=false``.  Host C++ (the C ABI) is compiled with g++.  The
result links cuBLAS for the plain dense GEMMs and nothing else.

Usage: ``python -m paper_2506_03275_b200.build [--force] [--verbose]``
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libcsd_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-I", INCLUDE, "-I", CSRC, "--expt-relaxed-constexpr"]
PER_FILE = {
    # bit-exact reference arithmetic: no FMA contraction, IEEE div/sqrt, denormals kept
    # debug timelines compiled out of the production build (CSD_TRACE=1 builds them in): the
    # predicated stamps cost 4 us of instruction fetch in the CTA-pair attention kernel
    "attn_cp.cu": [] if os.environ.get("CSD_TRACE") else ["-DCSD_CP_NOTRACE"],
    "attn_pp.cu": [] if os.environ.get("CSD_TRACE") else ["-DCSD_PP_NOTRACE"],
    "attn_sd.cu": [] if os.environ.get("CSD_TRACE") else ["-DCSD_SD_NOTRACE"],
    "check_kernels.cu": ["-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false"],
    # the CHECK latent update is the reference's separate multiply and add
    "generation.cu": ["-fmad=false"],
}
CXX_FLAGS = ["-O2", "-fPIC", "-std=c++17", "-I", INCLUDE, "-I", CSRC,
             "-I", os.path.join(CUDA, "include")]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE) if f.endswith(".h")]
    return max(os.path.getmtime(h) for h in hs)


def _compile(src, force, verbose):
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(path), _headers_mtime())):
        return obj, None
    if src.endswith(".cu"):
        cmd = [NVCC] + CU_FLAGS + PER_FILE.get(src, []) + ["-c", path, "-o", obj]
    else:
        cmd = ["g++"] + CXX_FLAGS + ["-c", path, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, f"{src}:\n{r.stdout}\n{r.stderr}"
    if verbose and r.stderr.strip():
        print(r.stderr, flush=True)
    return obj, None


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose), srcs))
    errs = [e for _, e in results if e]
    if errs:
        raise RuntimeError("CUDA build failed:\n" + "\n".join(errs))
    objs = [o for o, _ in results]
    if (force or not os.path.exists(LIB)
            or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs)):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-L", os.path.join(CUDA, "lib64"), "-lcublas",
            "-Xlinker", "-rpath," + os.path.join(CUDA, "lib64")]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_host(force, verbose)
    return LIB


HOST_SRC = os.path.join(PKG, "host", "csd_host.cpp")
HOST_LIB = os.path.join(PKG, "libcsd_host.so")


def build_host(force: bool = False, verbose: bool = False) -> str:
    """libcsd_host.so: the reference's C++ csd:: API (include/csd/*.hpp) over the C ABI."""
    deps = [HOST_SRC, LIB] + [os.path.join(INCLUDE, "csd", f)
                              for f in os.listdir(os.path.join(INCLUDE, "csd"))]
    if (not force and os.path.exists(HOST_LIB)
            and os.path.getmtime(HOST_LIB) >= max(os.path.getmtime(p) for p in deps)):
        return HOST_LIB
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
           "-I", INCLUDE, "-o", HOST_LIB, HOST_SRC,
           "-L", PKG, "-l:libcsd_b200.so", "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"host library build failed:\n{r.stdout}\n{r.stderr}")
    return HOST_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
