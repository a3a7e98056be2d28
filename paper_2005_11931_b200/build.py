"""Build libtsw.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", "tsw_runtime.cu")]
DEPS = SRC + [os.path.join(PKG, "csrc", "tsw_kernels.cuh"), os.path.join(ROOT, "include", "tsw.h")]
LIB = os.path.join(PKG, "libtsw.so")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "--fmad=false",            # no FMA contraction anywhere (R19); the stepper also uses __d*_rn
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-O2",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines: tuple = ()) -> str:
    """Compile libtsw.so if any source is newer than it.  Returns its path.

    `out` / `defines` build an alternative library (e.g. `-DTSW_TB_F32X2=0`) for A/B timing
    through the TSW_LIB override; the default build is the product.
    """
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return out
    cmd = [nvcc(), *NVCC_FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp", *SRC, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libtsw.so")
    if out == LIB:
        with open(os.path.join(PKG, "build_ptxas.log"), "w") as f:
            f.write(r.stderr)
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    # python -m paper_2005_11931_b200.build [--force] [--verbose] [--out PATH] [-DNAME=V ...]
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else LIB
    print(build(force="--force" in argv, verbose="--verbose" in argv, out=out,
                defines=tuple(a for a in argv if a.startswith("-D"))))
