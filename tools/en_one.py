"""One fused-energy pass of depth K on the bench workload (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2005_11931_b200 import inputs, tsw

dtype, K = sys.argv[1], int(sys.argv[2])
cfg = inputs.weak_unit(1)
s = tsw.Solver.from_config(cfg, dtype)
s.set_option(tsw.TSW_OPT_TBLOCK, K)
s.set_initial(inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(np.float64 if dtype == "f64" else np.float32),
              None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
s.step(1)
s.set_option(tsw.TSW_OPT_ENERGY_FUSE, 0)
s.step(K)          # plain pass
s.set_option(tsw.TSW_OPT_ENERGY_FUSE, 1)
s.step(K)          # fused pass
print(s.energy())
