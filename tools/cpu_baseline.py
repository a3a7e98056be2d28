#!/usr/bin/env python
"""The CPU oracle as a baseline on this host: full runs of configs 1–3 and prefixes
of configs 4 / 5, at all cores and at one core, one JSON line each (point-updates per second).
The oracle is test infrastructure: this tool only times it, as it stands.  Config 4's 32768² grid
is timed on a full-width band (the dense face arrays of the whole grid would not fit host memory
next to it); config 5 on a subset of members (each member is an independent grid)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import oracle
from paper_2005_11931_b200 import inputs


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def timed_run(cfg, member, dtype, nsteps, u0, rows=None):
    """Oracle start-up + nsteps−1 leapfrog levels of one member (optionally a full-width row band)."""
    npdt = np.float64 if dtype == "f64" else np.float32
    if rows is None:
        _, _, c1, c2 = oracle.member_coefficients(cfg, member, npdt)
        u = np.ascontiguousarray(u0, dtype=npdt)
    else:
        j0 = cfg.ny // 2 - rows // 2
        _, _, c1, c2 = oracle.member_coefficients(cfg, member, npdt, 0, j0, cfg.nx, rows)
        u = np.ascontiguousarray(u0(j0, rows), dtype=npdt)
    t = time.perf_counter()
    oracle.run(cfg.dim, c1, c2, u, None, cfg.dt, nsteps)
    el = time.perf_counter() - t
    ny = 1 if cfg.dim == 1 else u.shape[0]
    upd = (cfg.nx - 2) * max(ny - 2, 1) * nsteps
    return upd, el


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    lines = []
    ncores = cores()
    plan = [
        # (name, cfg, members, dtype, steps all-core, steps one-core, band rows)
        ("config1", inputs.config(1), [0], "f64", 4000, 4000, None),
        ("config1", inputs.config(1), [0], "f32", 4000, 4000, None),
        ("config2", inputs.config(2), [0, 1, 2, 3], "f64", 5000, 500, None),
        ("config3", inputs.config(3), [0], "f64", 5000, 50, None),
        ("config3", inputs.config(3), [0], "f32", 5000, 50, None),
        ("config4", inputs.config(4), [0], "f64", 20, 4, 4096),
        ("config5", inputs.config(5), [0, 31, 63, 64], "f64", 200, 20, None),
    ]
    for name, cfg, members, dtype, s_all, s_one, band in plan:
        for threads, steps, mem in ((ncores, s_all, members), (1, s_one, members[:1])):
            oracle.set_threads(threads)
            if band:
                u0 = lambda j0, rows: inputs.uniform_dense_rows(cfg.nx, cfg.ny, j0, rows)
            elif cfg.name.startswith("config4"):
                u0 = None
            else:
                u0 = cfg.initial()
            upd = el = 0.0
            for b in mem:
                u, e = timed_run(cfg, b, dtype, steps, u0, band)
                upd += u
                el += e
            line = {"config": name, "dtype": dtype, "threads": threads, "members": len(mem), "steps": steps,
                    "sample": ("full run" if steps == cfg.nsteps and not band else
                               f"{steps} of {cfg.nsteps} levels" + (f", {band}-row full-width band" if band else "")),
                    "updates": upd, "seconds": el, "gupd_per_s": upd / el / 1e9}
            print(json.dumps(line), flush=True)
            lines.append(line)
    if out:
        with open(out, "w") as f:
            for l in lines:
                f.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()
