"""In-tree build of the native library ``libhfmm_b200.so`` (sm_100a only).

The shared library holds the host setup (C++), the CUDA engine and the C ABI
declared in ``include/hfmm_gpu.h``.  It is built in-tree so it travels to the
GPU box with the repository snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2006_15367_b200")
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libhfmm_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["setup.cpp", "setup_import.cpp", "setup_gpu.cu", "engine.cu", "world.cu", "capi.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h")))


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libhfmm_b200.so")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    """Compiles the native library if any source changed; returns its path."""
    os.makedirs(os.path.join(OUT_DIR, "obj"), exist_ok=True)
    nvcc = _nvcc()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "hfmm_gpu.h")]
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OUT_DIR, "obj", src + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [path] + hdrs):
            continue
        if src.endswith(".cu"):
            cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v", *inc, "-c", path, "-o", obj]
        else:
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-pthread", *inc,
                   "-I", "/usr/local/cuda/include", "-c", path, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if verbose and res.stderr:
            print(res.stderr, file=sys.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"compile failed for {src}:\n{res.stdout}\n{res.stderr}")
    if force or _stale(LIB, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-pthread"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return LIB


def build_oracle(verbose: bool = False) -> str | None:
    """Builds oracle/_ref/libhfmm_ref.so from /root/reference (test checker only).

    Returns the library path, or None when the reference sources are absent
    (the GPU box uses the prebuilt file that travels with the snapshot).
    """
    lib = os.path.join(ROOT, "oracle", "_ref", "libhfmm_ref.so")
    if not os.path.isdir("/root/reference/proj/src"):
        return lib if os.path.exists(lib) else None
    res = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8"],
                         capture_output=True, text=True)
    if verbose:
        print(res.stdout[-2000:], res.stderr[-2000:], file=sys.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout[-4000:]}\n{res.stderr[-4000:]}")
    return lib


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
    print(build_oracle(verbose=True))
