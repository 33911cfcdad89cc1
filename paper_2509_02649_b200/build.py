"""Build libfk.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2509_02649_b200.build [--force]

Every .cu under csrc/ is compiled to an object with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked with cuFFT and cuSOLVER
into ``paper_2509_02649_b200/libfk.so``.  The seeded data generator (datagen/gen.cu, not part of
the method) is built alongside into ``datagen/libfkgen.so``.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfk.so")
GEN_SRC = os.path.join(ROOT, "datagen", "gen.cu")
GEN_LIB = os.path.join(ROOT, "datagen", "libfkgen.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, obj: str, verbose: bool) -> str:
    cmd = [NVCC] + FLAGS + ["-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return r.stderr if verbose else ""


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "fk.h")]
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    if force or _stale(LIB, srcs + hdrs):
        objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]
        with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
            logs = list(ex.map(lambda so: _compile(so[0], so[1], verbose), zip(srcs, objs)))
        if verbose:
            for l in logs:
                sys.stderr.write(l)
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + [
            "-L", os.path.join(CUDA, "lib64"), "-lcufft", "-lcusolver", "-lcublas",
            "-Xlinker", "-rpath=" + os.path.join(CUDA, "lib64")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr)
        os.replace(tmp, LIB)
    if force or _stale(GEN_LIB, [GEN_SRC]):
        tmp = GEN_LIB + f".tmp{os.getpid()}"
        cmd = [NVCC] + ARCH + ["-O3", "-Xcompiler", "-fPIC", "-shared", "-o", tmp, GEN_SRC]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for datagen/gen.cu:\n" + r.stderr)
        os.replace(tmp, GEN_LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
