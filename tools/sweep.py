"""Sweep stencil variants / ring shapes on the bench workload and print kernel GB/s (GPU only)."""
import argparse
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--depths", default="4,6,8,12")
    ap.add_argument("--warps", default="0")
    ap.add_argument("--rows", default="0")
    ap.add_argument("--nx", type=int, default=32768)
    ap.add_argument("--ny", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--kind", type=int, default=1)
    ap.add_argument("--reg", action="store_true", help="also time the register kernel")
    ap.add_argument("--tblocks", default="", help="temporal blocking depths to time, e.g. 2,4,8")
    ap.add_argument("--tbdepths", default="4")
    args = ap.parse_args()
    import torch
    from paper_2005_11931_b200 import inputs, tsw
    cfg = inputs.config(4, nx=args.nx, ny=args.ny, kind=args.kind, eps=[0.05] * args.batch,
                        amp=[1.0] * args.batch)
    esz = 8 if args.dtype == "f64" else 4
    npdt = np.float64 if args.dtype == "f64" else np.float32
    s = tsw.Solver.from_config(cfg, args.dtype)
    u0 = inputs.uniform_dense((cfg.ny, cfg.nx), seed=0).astype(npdt)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(100)
    combos = [(0, d, w, r) for d, w, r in itertools.product(
        [int(x) for x in args.depths.split(",")], [int(x) for x in args.warps.split(",")],
        [int(x) for x in args.rows.split(",")])]
    if args.reg:
        combos = [(1, 0, 0, r) for r in [int(x) for x in args.rows.split(",")]] + combos
    for K in [int(x) for x in args.tblocks.split(",") if x]:
        for td in [int(x) for x in args.tbdepths.split(",")]:
            for r in [int(x) for x in args.rows.split(",")]:
                s.set_option(tsw.TSW_OPT_TBLOCK, K)
                s.set_option(tsw.TSW_OPT_TB_DEPTH, td)
                s.set_option(tsw.TSW_OPT_ROWS_PER_ITEM, r)
                try:
                    s.step(4 * K)
                    s.set_option(tsw.TSW_OPT_TIME_KERNELS, 1)
                    s.step((args.steps // K) * K)
                    ms, n, upd = s.kernel_stats()
                    s.set_option(tsw.TSW_OPT_TIME_KERNELS, 0)
                except tsw.TswError as e:
                    print(json.dumps({"tblock": K, "tbdepth": td, "rows": r, "error": str(e)}), flush=True)
                    continue
                print(json.dumps({"kernel": "tb", "K": K, "tbdepth": td, "rows": r, "ms_per_level": ms / (n * K),
                                  "Gpts": round(upd / (ms * 1e-3) / 1e9, 2),
                                  "hbm_GBs_4words_per_pass": round(upd / K * 4 * esz / (ms * 1e-3) / 1e9, 1)}),
                      flush=True)
        s.set_option(tsw.TSW_OPT_TBLOCK, 1)
    for kern, d, w, r in combos:
        s.set_option(tsw.TSW_OPT_KERNEL, kern)
        if kern == 0:
            s.set_option(tsw.TSW_OPT_DEPTH, d)
        s.set_option(tsw.TSW_OPT_ROWS_PER_ITEM, r)
        try:
            s.step(20)
            s.set_option(tsw.TSW_OPT_TIME_KERNELS, 1)
            s.step(args.steps)
            ms, n, upd = s.kernel_stats()
            s.set_option(tsw.TSW_OPT_TIME_KERNELS, 0)
        except tsw.TswError as e:
            print(json.dumps({"kernel": kern, "depth": d, "warps": w, "rows": r, "error": str(e)}))
            continue
        gbs = upd * 3 * esz / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": "tma" if kern == 0 else "reg", "depth": d, "warps": w, "rows": r,
                          "ms_per_launch": ms / n, "GBs": round(gbs, 1), "Gpts": round(upd / (ms * 1e-3) / 1e9, 2)}),
              flush=True)


if __name__ == "__main__":
    main()
