"""Interleaved A/B of the temporally blocked stencil's CTA width (4 vs 8 warps) on config 3 / 5."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def main():
    from paper_2005_11931_b200 import inputs, tsw
    which, dtype = sys.argv[1], sys.argv[2]
    K = 4 if dtype == "f64" else 8
    cfg = inputs.config(5) if which == "config5" else inputs.config(3)
    npdt = np.float64 if dtype == "f64" else np.float32
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_initial(cfg.initial().astype(npdt), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(1)
    s.set_option(tsw.TSW_OPT_TBLOCK, K)
    res = {4: [], 8: []}
    for rep in range(4):
        for w in (4, 8):
            s.set_option(tsw.TSW_OPT_TB_WARPS, w)
            s.step(4 * K)
            s.set_option(tsw.TSW_OPT_TIME_KERNELS, 1)
            s.step(24 * K)
            ms, n, upd = s.kernel_stats()
            s.set_option(tsw.TSW_OPT_TIME_KERNELS, 0)
            res[w].append(round(upd / (ms * 1e-3) / 1e9, 1))
    print(json.dumps({"workload": which, "dtype": dtype, "w4": res[4], "w8": res[8],
                      "w4_median": float(np.median(res[4])), "w8_median": float(np.median(res[8]))}))


if __name__ == "__main__":
    main()
