#!/usr/bin/env python
"""Paper Table 1 workload on the implicit scheme (TSW_OPT_SCHEME = 1): H = h_0(x),
ε = 0.8, Gaussian u0 on [0,100]², N² nodes, 100 steps of Δt = 0.05.  Times the 100 levels with
CUDA events (start-up level included, coefficient build excluded) and prints one JSON line per
size and dtype; `--kernels` adds a per-kernel breakdown from torch.profiler-free event timing of
one isolated level of each kernel class (run separately, never under ncu)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_2005_11931_b200 import inputs, tsw

PAPER_GPU_S = {256: 0.88, 512: 2.07, 1024: 7.16, 2048: 20.30, 4096: 62.76}
PAPER_CPU_S = {256: 0.91, 512: 3.73, 1024: 15.92, 2048: 64.8, 4096: 280.54}


def run(n, dtype, steps, reps, solver=0, xrows=1):
    sc = inputs.paper_2d(dx=100.0 / (n - 1))
    assert sc.nx == n and sc.ny == n, (sc.nx, sc.ny)
    stream = torch.cuda.Stream()
    s = tsw.Solver(2, n, n, sc.dx, sc.dx, 1, dtype, stream=stream.cuda_stream)
    s.set_coeff_profile(sc.seg_value, sc.seg_break, [0.8], isotropic=True)
    s.set_option(tsw.TSW_OPT_SCHEME, 1)
    s.set_option(tsw.TSW_OPT_IMPLICIT_SOLVER, solver)
    s.set_option(tsw.TSW_OPT_IMPLICIT_XROWS, xrows)
    u0 = sc.initial().astype(np.float64 if dtype == "f64" else np.float32)[None]
    u0d = torch.from_numpy(u0).cuda()
    best = None
    for r in range(reps + 1):
        s.set_initial(u0d, None, 0.05)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = s.launches()
        e0.record(stream)
        s.step(steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if r > 0:                           # first repetition = warm-up
            best = ms if best is None else min(best, ms)
        launches = s.launches() - l0
    g = s.read(0)[0]
    s.close()
    return best, launches, float(np.max(np.abs(g)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="256,512,1024,2048,4096")
    ap.add_argument("--dtypes", default="f64,f32")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--xrows", type=int, default=1)
    ap.add_argument("--solver", type=int, default=0, help="TSW_OPT_IMPLICIT_SOLVER (0 cluster scans, 1 CR, 2 streaming scans)")
    args = ap.parse_args()
    for dtype in args.dtypes.split(","):
        for n in [int(x) for x in args.sizes.split(",")]:
            ms, launches, umax = run(n, dtype, args.steps, args.reps, args.solver, args.xrows)
            esz = 8 if dtype == "f64" else 4
            line = {"workload": f"table1_implicit_{n}x{n}", "dtype": dtype, "solver": args.solver, "xrows": args.xrows, "steps": args.steps, "ms": ms,
                    "mpts": n * n * args.steps / (ms * 1e-3) / 1e6, "launches": launches, "max_abs_u": umax,
                    "paper_gpu_s": PAPER_GPU_S.get(n), "paper_cpu_s": PAPER_CPU_S.get(n),
                    "speedup_vs_paper_gpu": (PAPER_GPU_S[n] * 1e3 / ms) if n in PAPER_GPU_S else None,
                    "hbm_gbs_at_9_words": n * n * args.steps * 9 * esz / (ms * 1e-3) / 1e9}
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
