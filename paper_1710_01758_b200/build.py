"""Build libsbpcg.so (sm_100a) in-tree with nvcc.  `python -m paper_1710_01758_b200.build`."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libsbpcg.so")
SOURCES = ["sbpcg.cu", "k_matvec.cu", "k_passes.cu", "k_lambda.cu", "k_sb.cu", "k_plane.cu", "k_plane3.cu", "k_coil.cu", "k_prep.cu", "k_wav.cu", "k_persist.cu"]
HEADERS = ["fft_core.cuh", "internal.cuh", "kernels.cuh", "pcg_fin.cuh", "sb_tile.cuh", "k_plane.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v" if os.environ.get("SBPCG_PTXAS_V") else "-O3",
    "-I" + os.path.join(os.path.dirname(HERE), "include"),
]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def _compile(src):
    s = os.path.join(CSRC, src)
    o = os.path.join(OBJ, src.replace(".cu", ".o"))
    deps = [s] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(os.path.dirname(HERE), "include", "sbpcg.h")]
    if os.path.exists(o) and os.path.getmtime(o) >= _newest(deps):
        return o, ""
    cmd = [NVCC, *FLAGS, "-dc" if False else "-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return o, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
               *objs, "-ldl", "-o", LIB]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
