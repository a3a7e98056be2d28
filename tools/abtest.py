"""Interleaved A/B timing of temporal-blocking depths on the bench workload (GPU only)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def main():
    import torch
    from paper_2005_11931_b200 import inputs, tsw
    dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
    Ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,5").split(",")]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    cfg = inputs.weak_unit(1)
    npdt = np.float64 if dtype == "f64" else np.float32
    s = tsw.Solver.from_config(cfg, dtype)
    if os.environ.get("TSW_AB_WARPS"):   # CTA width of the TB stencil (TSW_OPT_TB_WARPS)
        s.set_option(tsw.TSW_OPT_TB_WARPS, int(os.environ["TSW_AB_WARPS"]))
    if os.environ.get("TSW_AB_DEPTH"):   # input ring stages (TSW_OPT_TB_DEPTH)
        s.set_option(tsw.TSW_OPT_TB_DEPTH, int(os.environ["TSW_AB_DEPTH"]))
    s.set_initial(inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(npdt), None, cfg.dt,
                  flags=tsw.TSW_INIT_SHARED)
    s.step(1)
    res = {K: [] for K in Ks}
    for rep in range(reps):
        for K in Ks:
            s.set_option(tsw.TSW_OPT_TBLOCK, K)
            s.step(8 * K)
            s.set_option(tsw.TSW_OPT_TIME_KERNELS, 1)
            s.step(40 * K)
            ms, n, upd = s.kernel_stats()
            s.set_option(tsw.TSW_OPT_TIME_KERNELS, 0)
            res[K].append(upd / (ms * 1e-3) / 1e9)
    print(json.dumps({"dtype": dtype, **{f"K{K}": [round(x, 1) for x in v] for K, v in res.items()},
                      **{f"K{K}_median": round(float(np.median(v)), 1) for K, v in res.items()}}))


if __name__ == "__main__":
    main()
