"""Cost of the slab decomposition on one GPU: P loopback slabs of the bench's weak unit stepped
with tsw_group_step (split passes: boundary rows first, K-row exchanges) against one domain of the
same total rows.  Prints one JSON line.  python tools/slab_overhead.py [f64|f32] [K] [P] [peer]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def main():
    import torch
    from paper_2005_11931_b200 import inputs, tsw
    dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    P = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    peer = len(sys.argv) > 4 and sys.argv[4] == "peer"
    npdt = np.float64 if dtype == "f64" else np.float32
    cfg = inputs.weak_unit(P)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(npdt)
    stream = torch.cuda.Stream()
    n = 10 * K

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    one = tsw.Solver.from_config(cfg, dtype, stream=stream.cuda_stream)
    one.set_option(tsw.TSW_OPT_TBLOCK, K)
    one.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    one.step(1 + K)
    t_one = min(timed(lambda: one.step(n)) for _ in range(3))
    one.close()
    # the weak-scaling reference: one slab's rows as a single domain (the N = 1 bench run), × P
    c1 = inputs.weak_unit(1)
    u1 = np.ascontiguousarray(u0[:c1.ny])
    unit = tsw.Solver.from_config(c1, dtype, stream=stream.cuda_stream)
    unit.set_option(tsw.TSW_OPT_TBLOCK, K)
    unit.set_initial(u1, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    unit.step(1 + K)
    t_unit = P * min(timed(lambda: unit.step(n)) for _ in range(3))
    unit.close()
    parts = [tsw.Solver.from_config(cfg, dtype, rank=r, nranks=P, stream=stream.cuda_stream) for r in range(P)]
    for p in parts:
        p.set_option(tsw.TSW_OPT_TBLOCK, K)
    if peer:
        for p in parts:
            p.set_option(tsw.TSW_OPT_HALO, 1)
        for r, p in enumerate(parts):
            if r > 0:
                p.peer_attach(0, parts[r - 1])
            if r < P - 1:
                p.peer_attach(1, parts[r + 1])
    for p in parts:
        p.set_initial(np.ascontiguousarray(u0[p.r0:p.r0 + p.ny_local]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    ctxs = [p.ctx for p in parts]
    tsw.tsw_group_step(ctxs, 1 + K)
    t_grp = min(timed(lambda: tsw.tsw_group_step(ctxs, n)) for _ in range(3))
    for p in parts:
        p.close()
    print(json.dumps({"dtype": dtype, "K": K, "P": P, "peer": peer, "levels": n, "ms_one_domain": round(t_one, 3),
                      "ms_slabs": round(t_grp, 3), "overhead": round(t_grp / t_one - 1, 4),
                      "ms_P_x_unit": round(t_unit, 3), "overhead_vs_unit": round(t_grp / t_unit - 1, 4)}))


if __name__ == "__main__":
    main()
