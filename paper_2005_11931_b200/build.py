"""Build libtsw.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# translation units: the runtime (all other kernels) and the temporally blocked stencil's launch
# wrappers once per precision and variant (plain / fused energy) — compiled in parallel, then
# linked into one shared library
UNITS = [("tsw_runtime", "tsw_runtime.cu", ()),
         ("tsw_tb_f64", "tsw_tb.cu", ("-DTSW_TB_DTYPE=double", "-DTSW_TB_EN=0")),
         ("tsw_tb_f64_en", "tsw_tb.cu", ("-DTSW_TB_DTYPE=double", "-DTSW_TB_EN=1")),
         ("tsw_tb_f32", "tsw_tb.cu", ("-DTSW_TB_DTYPE=float", "-DTSW_TB_EN=0")),
         ("tsw_tb_f32_en", "tsw_tb.cu", ("-DTSW_TB_DTYPE=float", "-DTSW_TB_EN=1"))]
SRC = [os.path.join(CSRC, u[1]) for u in UNITS]
DEPS = sorted(set(SRC)) + [os.path.join(CSRC, "tsw_kernels.cuh"), os.path.join(ROOT, "include", "tsw.h")]
LIB = os.path.join(PKG, "libtsw.so")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "--fmad=false",            # no FMA contraction anywhere (R19); the stepper also uses __d*_rn
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-O2",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines: tuple = ()) -> str:
    """Compile libtsw.so if any source is newer than it.  Returns its path.

    `out` / `defines` build an alternative library (e.g. `-DTSW_TB_SHFL_F64=0`) for A/B timing
    through the TSW_LIB override; the default build is the product.
    """
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return out
    objdir = out + ".obj"
    os.makedirs(objdir, exist_ok=True)
    procs = []
    for name, src, extra in UNITS:
        obj = os.path.join(objdir, name + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *extra, *defines, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj,
               os.path.join(CSRC, src)]
        procs.append((name, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    logs, objs, failed = [], [], []
    for name, obj, p in procs:
        so, se = p.communicate()
        logs.append(f"==== {name}\n{se}")
        objs.append(obj)
        if p.returncode != 0:
            failed.append(name)
            sys.stderr.write(so + se)
    if failed:
        raise RuntimeError(f"nvcc failed building {failed}")
    r = subprocess.run([nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out + ".tmp", *objs,
                        "-ldl"], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libtsw.so")
    if out == LIB:
        with open(os.path.join(PKG, "build_ptxas.log"), "w") as f:
            f.write("".join(logs))
    if verbose:
        sys.stderr.write("".join(logs))
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    # python -m paper_2005_11931_b200.build [--force] [--verbose] [--out PATH] [-DNAME=V ...]
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else LIB
    print(build(force="--force" in argv, verbose="--verbose" in argv, out=out,
                defines=tuple(a for a in argv if a.startswith("-D"))))
