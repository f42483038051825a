"""In-tree build of libsk_cuda.so (sm_100a) with nvcc.

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box; objects go to build/. No JIT cache is used.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libsk_cuda.so"

SOURCES = ["sk_common.cu", "sk_stencil.cu", "sk_ch.cu", "sk_blas.cu", "sk_csr.cu", "sk_cg.cu", "sk_imex.cu", "sk_spectral.cu", "sk_matmul.cu", "sk_refine.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    f"-I{ROOT / 'include'}",
    f"-I{CSRC}",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libsk_cuda.so")


def _newest_input() -> float:
    files = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp"))
    files += [ROOT / "include" / "sk_cuda.h", Path(__file__)]
    return max(f.stat().st_mtime for f in files)


def _compile(src: str) -> tuple[str, str]:
    obj = BUILD / (Path(src).stem + ".o")
    cmd = [nvcc(), *NVCC_FLAGS, "-c", str(CSRC / src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    (BUILD / (Path(src).stem + ".ptxas.log")).write_text(res.stderr)
    return src, res.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every CUDA source for sm_100a and link libsk_cuda.so in-tree."""
    if not force and LIB.exists() and LIB.stat().st_mtime >= _newest_input():
        return LIB
    BUILD.mkdir(exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        for src, log in ex.map(_compile, SOURCES):
            if verbose:
                print(f"[nvcc] {src}\n{log}", file=sys.stderr)
    objs = [str(BUILD / (Path(s).stem + ".o")) for s in SOURCES]
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


def build_oracle() -> None:
    """Build the CPU checker (oracle/, test infrastructure only)."""
    env = dict(os.environ)
    res = subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "-j8"], capture_output=True, text=True, env=env)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout}\n{res.stderr}")


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_oracle()
    print(LIB)
