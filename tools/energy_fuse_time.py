"""Fused-energy pass vs plain pass on the bench workload (GPU only): per-launch CUDA-event times of
one K-level pass with TSW_OPT_ENERGY_FUSE on / off, interleaved, plus the standalone energy call."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def main():
    from paper_2005_11931_b200 import inputs, tsw
    dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
    Ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "8,4").split(",")]
    cfg = inputs.weak_unit(1)
    npdt = np.float64 if dtype == "f64" else np.float32
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_option(tsw.TSW_OPT_TBLOCK, max(Ks))
    s.set_initial(inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(npdt), None, cfg.dt,
                  flags=tsw.TSW_INIT_SHARED)
    s.step(17)
    out = {"dtype": dtype}
    for K in Ks:
        s.set_option(tsw.TSW_OPT_TBLOCK, K)
        res = {0: [], 1: []}
        for rep in range(6):
            for fuse in (0, 1):
                s.set_option(tsw.TSW_OPT_ENERGY_FUSE, fuse)
                s.set_option(tsw.TSW_OPT_TIME_KERNELS, 1)
                s.step(K)
                ms, lv, up = s.kernel_launches()
                s.set_option(tsw.TSW_OPT_TIME_KERNELS, 0)
                res[fuse].append(float(ms[-1]))
        # end-to-end: step(K) + energy(), fused vs standalone, wall time over 10 repetitions
        e2e = {}
        for fuse in (0, 1):
            s.set_option(tsw.TSW_OPT_ENERGY_FUSE, fuse)
            s.sync()
            t = time.perf_counter()
            for _ in range(10):
                s.step(K)
                s.energy()
            e2e[fuse] = (time.perf_counter() - t) / 10 * 1e3
        out[f"K{K}"] = {"plain_ms": float(np.median(res[0])), "fused_ms": float(np.median(res[1])),
                        "overhead": float(np.median(res[1]) / np.median(res[0]) - 1),
                        "step_plus_energy_ms_standalone": e2e[0], "step_plus_energy_ms_fused": e2e[1]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
