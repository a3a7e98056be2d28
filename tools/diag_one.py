"""One standalone energy and one second-wave call on config 5 (65 × 2048², for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2005_11931_b200 import inputs, tsw

dtype = sys.argv[1] if len(sys.argv) > 1 else "f32"
cfg = inputs.config(5)
s = tsw.Solver.from_config(cfg, dtype)
s.set_initial(cfg.initial().astype(np.float64 if dtype == "f64" else np.float32), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
s.set_option(tsw.TSW_OPT_ENERGY_FUSE, 0)
s.step(3)
print(s.energy()[0], s.wave2(cfg.batch - 1)[0])
