"""In-tree build of the sm_100a CUDA library (libternary_b200.so).

Plain nvcc, one object per .cu, linked as a shared library next to the
Python package so it travels to the GPU box with the repo snapshot:

    python -m paper_2410_16144_b200.build
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "lib"
LIB = OUT_DIR / "libternary_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr"]
SOURCES = ["abi.cu", "quantize.cu", "pack.cu", "gemv.cu", "gemv_aux.cu", "gemm_tc.cu",
           "allreduce.cu"]


def _sources():
    return [CSRC / s for s in SOURCES if (CSRC / s).exists()]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "ternary_b200.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps if d.exists())


def _compile(src: Path, obj: Path, verbose: bool) -> None:
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)


def build(force: bool = False, verbose: bool = False) -> Path:
    OUT_DIR.mkdir(exist_ok=True)
    objs = []
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for src in _sources():
            obj = OUT_DIR / (src.stem + ".o")
            objs.append(obj)
            if force or _stale(obj, src):
                jobs.append(ex.submit(_compile, src, obj, verbose))
        for j in jobs:
            j.result()
    if force or jobs or not LIB.exists():
        cmd = [NVCC, *ARCH, "-shared", *map(str, objs), "-o", str(LIB), "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
