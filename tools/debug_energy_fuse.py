"""Debug: fused vs standalone energy over shapes / CTA widths / rows per item (GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2005_11931_b200 import inputs, tsw

for (ny, nx) in [(97, 700), (300, 2049), (64, 300), (40, 1100)]:
    for warps in (4, 8):
        for rpi in (0, 1000, 7):
            for K in (8, 4):
                cfg = inputs.config(3, nx=nx, ny=ny, dx=0.01, dy=0.01, eps=[0.1], amp=[1.0], dt=2e-3)
                u0 = inputs.uniform_dense_rows(nx, ny, 0, ny)
                s = tsw.Solver.from_config(cfg, "f64")
                s.set_option(tsw.TSW_OPT_TBLOCK, K)
                s.set_option(tsw.TSW_OPT_TB_WARPS, warps)
                if rpi:
                    s.set_option(tsw.TSW_OPT_ROWS_PER_ITEM, rpi)
                s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
                s.step(1)
                s.step(K)
                Ef = s.energy()[0]
                s.set_option(tsw.TSW_OPT_ENERGY_FUSE, 0)
                Es = s.energy()[0]
                print(f"ny={ny} nx={nx} warps={warps} rpi={rpi} K={K}: rel {(Ef - Es) / Es:+.3e}  diff {Ef - Es:+.6e}",
                      flush=True)
                s.close()
