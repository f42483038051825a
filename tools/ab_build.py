#!/usr/bin/env python3
"""Build an alternative libsk_cuda.so for same-box A/B timing (tools only).

    python tools/ab_build.py <name> [--rev GIT_REV] [-DMACRO=V ...]

Compiles the CUDA sources of the working tree (or of git revision REV) with
optional extra -D flags into _ab/<name>.so (git-ignored; travels to the GPU
box with the snapshot). Timing tools load it with `--lib _ab/<name>.so`;
the product loader (_lib.load) never looks there on its own.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2205_03354_b200 import build_ext  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--rev", default=None)
    args, extra = ap.parse_known_args()
    out = ROOT / "_ab" / f"{args.name}.so"
    out.parent.mkdir(exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        if args.rev:
            tar = subprocess.run(["git", "-C", str(ROOT), "archive", args.rev, "paper_2205_03354_b200/csrc", "include"],
                                 check=True, capture_output=True).stdout
            subprocess.run(["tar", "-x", "-C", str(td)], input=tar, check=True)
            csrc, inc = td / "paper_2205_03354_b200" / "csrc", td / "include"
        else:
            csrc, inc = build_ext.CSRC, ROOT / "include"
        flags = build_ext.ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{inc}", f"-I{csrc}"]
        srcs = [s for s in build_ext.SOURCES if (csrc / s).exists()]

        def comp(src):
            obj = td / (Path(src).stem + ".o")
            r = subprocess.run([build_ext.nvcc(), *flags, *extra, "-c", str(csrc / src), "-o", str(obj)],
                               capture_output=True, text=True)
            if r.returncode:
                raise RuntimeError(r.stderr)
            return str(obj)

        with cf.ThreadPoolExecutor(len(srcs)) as ex:
            objs = list(ex.map(comp, srcs))
        subprocess.run([build_ext.nvcc(), *build_ext.ARCH, "-shared", "-o", str(out), *objs, "-lcudart_static", "-lrt",
                        "-ldl", "-lpthread"], check=True)
    print(out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
