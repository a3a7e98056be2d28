"""Time the diagnostics reductions (S5 energy, S6 second-wave amplitude, the ε-family L² distances)
on config 5's batch (65 × 2048², the workload that uses them) and on the bench slab; prints one JSON
line per case with the algorithmic bytes (fields read once) per second.
python tools/diag_time.py [f64|f32]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def med_ms(fn, reps=10):
    import torch
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        fn()
        t1.record()
        torch.cuda.synchronize()
        ts.append(t0.elapsed_time(t1))
    return float(np.median(ts))


def main():
    from paper_2005_11931_b200 import inputs, tsw
    dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
    esz = 8 if dtype == "f64" else 4
    npdt = np.float64 if dtype == "f64" else np.float32
    for name, cfg in (("config5", inputs.config(5)), ("bench_slab", inputs.weak_unit(1))):
        s = tsw.Solver.from_config(cfg, dtype)
        u0 = (cfg.initial() if name == "config5" else
              inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)).astype(npdt)
        s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
        s.step(3)
        field = cfg.batch * cfg.nx * cfg.ny * esz          # one level of every member
        out = {"dtype": dtype, "workload": name, "batch": cfg.batch, "nx": cfg.nx, "ny": cfg.ny}
        s.energy()
        ms = med_ms(s.energy)
        out["energy_ms"] = round(ms, 4)
        out["energy_GBs"] = round(2 * field / (ms * 1e-3) / 1e9, 1)        # reads u^n, u^{n-1}
        if cfg.batch > 1:
            s.wave2(cfg.batch - 1)
            ms = med_ms(lambda: s.wave2(cfg.batch - 1))
            out["wave2_ms"] = round(ms, 4)
            out["wave2_GBs"] = round(field / (ms * 1e-3) / 1e9, 1)         # reads u^n of every member
            s.family_l2()
            ms = med_ms(s.family_l2, reps=3)
            out["family_l2_ms"] = round(ms, 4)
            out["family_l2_GBs"] = round(field / (ms * 1e-3) / 1e9, 1)     # each member's field once
            # the roof that binds: fp64 instructions (a subtraction and a fused multiply-add per
            # member pair and node) against the measured fp64 add/multiply rate
            ops = cfg.batch * (cfg.batch - 1) / 2 * cfg.nx * cfg.ny * 2
            out["family_l2_TOPs"] = round(ops / (ms * 1e-3) / 1e12, 2)
            roof = tsw.tsw_alu_probe(0, tsw.TSW_F64)
            out["family_l2_alu_frac"] = round(ops / (ms * 1e-3) / roof, 3)
        s.close()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
