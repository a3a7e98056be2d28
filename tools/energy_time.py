"""Time tsw_energy (k_energy2d + k_energy_final) on the bench workload: python tools/energy_time.py [f64|f32]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def main():
    import torch
    from paper_2005_11931_b200 import inputs, tsw
    dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
    cfg = inputs.weak_unit(1)
    npdt = np.float64 if dtype == "f64" else np.float32
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_initial(inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(npdt), None, cfg.dt,
                  flags=tsw.TSW_INIT_SHARED)
    s.step(3)
    e = s.energy()
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        s.energy()
        t1.record()
        torch.cuda.synchronize()
        ts.append(t0.elapsed_time(t1))
    esz = 8 if dtype == "f64" else 4
    ms = float(np.median(ts))
    print(json.dumps({"dtype": dtype, "energy": float(e[0]), "ms_median": round(ms, 4),
                      "GBs_2_levels": round(2 * cfg.nx * cfg.ny * esz / (ms * 1e-3) / 1e9, 1)}))


if __name__ == "__main__":
    main()
