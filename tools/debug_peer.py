"""Step-by-step peer-halo group on one GPU with non-blocking progress checks (debugging)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2005_11931_b200 import inputs, tsw


def state(parts, streams, tag):
    print(tag, [tsw.tsw_peer_state(p.ctx) for p in parts], [s.query() for s in streams], flush=True)


def main():
    P, K = int(sys.argv[1]), int(sys.argv[2])
    cfg = inputs.config(3, nx=700, ny=151, dx=0.01, dy=0.01, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = [tsw.Solver.from_config(cfg, "f64", rank=r, nranks=P, stream=streams[r].cuda_stream) for r in range(P)]
    for p in parts:
        if K > 1:
            p.set_option(tsw.TSW_OPT_TBLOCK, K)
        p.set_option(tsw.TSW_OPT_HALO, 1)
    for r, p in enumerate(parts):
        if r > 0:
            p.peer_attach(0, parts[r - 1])
        if r < P - 1:
            p.peer_attach(1, parts[r + 1])
    state(parts, streams, "attached")
    for p in parts:
        p.set_initial(np.ascontiguousarray(u0[p.r0:p.r0 + p.ny_local]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
        state(parts, streams, f"init {p.rank}")
    time.sleep(1)
    state(parts, streams, "after init")
    for p in parts:
        p.step(1)
        state(parts, streams, f"step1 {p.rank}")
    time.sleep(1)
    state(parts, streams, "after step1")
    for p in parts:
        p.step(10)
    time.sleep(1)
    state(parts, streams, "after step10")
    print("reading", flush=True)
    print([float(np.abs(p.read(0)).max()) for p in parts], flush=True)


if __name__ == "__main__":
    main()
