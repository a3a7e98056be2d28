import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_11931_b200 import inputs, tsw
cfg = inputs.weak_unit(1)
u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
def mk(K, graphs=1):
    s = tsw.Solver.from_config(cfg, "f64")
    s.set_option(tsw.TSW_OPT_TBLOCK, K)
    s.set_option(tsw.TSW_OPT_GRAPHS, graphs)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    return s
r = mk(1, 0); r.step(41); ref = r.read(0)[0].copy(); r.close()
for mode in ("K1_graphs", "K1_nographs", "K4", "K1_graphs_concurrentTB", "K1_nographs_concurrentTB", "K4_concurrentTB"):
    fails = []
    for it in range(6):
        other = None
        if "concurrent" in mode:
            other = mk(4); other.step(41)      # async, still running
        K = 4 if mode.startswith("K4") else 1
        s = mk(K, 0 if "nographs" in mode else 1); s.step(41)
        g = s.read(0)[0]
        nb = int(np.sum(g != ref))
        if nb:
            rows = np.unique(np.argwhere(g != ref)[:, 0])
            fails.append((it, nb, int(rows.min()), int(rows.max()), len(rows)))
        s.close()
        if other: other.sync(); other.close()
    print(mode, "fails:", fails, flush=True)
