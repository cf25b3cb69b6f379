"""Builds libwr.so in-tree for sm_100a with nvcc (no JIT, no torch extension).

fp32 discipline (reading A6): -fmad=false (no FMA contraction), -ftz=false,
-prec-div/-prec-sqrt=true, no --use_fast_math.
"""
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libwr.so")
SOURCES = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HEADERS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "wr.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compiles each translation unit in parallel (no relocatable device
    code: every kernel lives in one .cu), then links libwr.so."""
    if force or needs_build():
        from concurrent.futures import ThreadPoolExecutor
        objdir = os.path.join(HERE, "build")
        os.makedirs(objdir, exist_ok=True)
        compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
        objs = [os.path.join(objdir, os.path.basename(src)[:-3] + ".o") for src in SOURCES]

        def one(pair):
            src, obj = pair
            cmd = [nvcc()] + compile_flags + ["-c", "-o", obj, src]
            if verbose:
                print(" ".join(cmd))
            subprocess.check_call(cmd)

        with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
            list(ex.map(one, zip(SOURCES, objs)))
        cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB] + objs
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
