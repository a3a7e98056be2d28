"""Exercise every kernel family on small grids (for compute-sanitizer memcheck / racecheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2005_11931_b200 import inputs, tsw


def main():
    # 1D config 1 (smem stepper), energy, wave2
    c1 = inputs.config(1, eps=[0.05, 0.2, 0.1], amp=[1.0, 1.0, 0.0])
    s = tsw.Solver.from_config(c1, "f64")
    s.set_initial(c1.initial(), None, c1.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(50)
    s.energy(); s.wave2(2); s.family_l2(); s.field_norms(); s.coeff_norms()
    s.close()
    for dtype in ("f64", "f32"):
        # 2D δ-point (dense faces), TMA and register kernels
        cfg = inputs.config(2, nx=200, ny=150, dx=0.01, dy=0.01, eps=[0.1, 0.2], amp=[1.0, 0.0], dt=3e-4)
        for kern in (0, 1):
            s = tsw.Solver.from_config(cfg, dtype)
            s.set_option(tsw.TSW_OPT_KERNEL, kern)
            s.set_initial(cfg.initial().astype(np.float64 if dtype == "f64" else np.float32), None, cfg.dt,
                          flags=tsw.TSW_INIT_SHARED)
            s.step(7)
            s.energy(); s.wave2(1); s.family_l2(); s.field_norms(); s.coeff_norms()
            s.close()
        # δ-line with temporal blocking
        cfg = inputs.config(3, nx=700, ny=97, dx=0.01, dy=0.01, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=2e-3)
        for K in (2, 4, 8):
            s = tsw.Solver.from_config(cfg, dtype)
            s.set_option(tsw.TSW_OPT_TBLOCK, K)
            s.set_option(tsw.TSW_OPT_ROWS_PER_ITEM, 20)
            s.set_initial(inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(
                np.float64 if dtype == "f64" else np.float32), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
            s.step(2 * K + 3)
            s.energy()
            s.close()
        # row slabs of one process: loopback copies (the NCCL pass's phases) and peer halos, with the
        # fused energy of the last pass
        import torch
        for halo in (0, 1):
            stream = torch.cuda.Stream()
            parts = [tsw.Solver.from_config(cfg, dtype, rank=r, nranks=2, stream=stream.cuda_stream) for r in range(2)]
            for p in parts:
                p.set_option(tsw.TSW_OPT_TBLOCK, 4)
                if halo:
                    p.set_option(tsw.TSW_OPT_HALO, 1)
            if halo:
                parts[0].peer_attach(1, parts[1])
                parts[1].peer_attach(0, parts[0])
            u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(np.float64 if dtype == "f64" else np.float32)
            for p in parts:
                p.set_initial(np.ascontiguousarray(u0[p.r0:p.r0 + p.ny_local]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
            tsw.tsw_group_step([p.ctx for p in parts], 1)
            tsw.tsw_group_step([p.ctx for p in parts], 11)
            for p in parts:
                p.energy()
                p.close()
        # profile coefficients + implicit (both solvers), 2D and 1D
        sc = inputs.paper_2d(dx=0.5)
        for solver in (0, 1):
            s = tsw.Solver(2, sc.nx, sc.ny, sc.dx, sc.dx, 1, dtype)
            s.set_coeff_profile(sc.seg_value, sc.seg_break, [0.8], isotropic=True)
            s.set_option(tsw.TSW_OPT_SCHEME, 1)
            s.set_option(tsw.TSW_OPT_IMPLICIT_SOLVER, solver)
            s.set_initial(sc.initial()[None].astype(np.float64 if dtype == "f64" else np.float32), None, 0.05)
            s.step(3)
            s.read(0)
            s.close()
        c1d = inputs.config(1, eps=[0.05], amp=[1.0], dt=0.02)
        s = tsw.Solver.from_config(c1d, dtype)
        s.set_option(tsw.TSW_OPT_SCHEME, 1)
        s.set_initial(c1d.initial().astype(np.float64 if dtype == "f64" else np.float32), None, c1d.dt,
                      flags=tsw.TSW_INIT_SHARED)
        s.step(3)
        s.close()
    print("ok")


if __name__ == "__main__":
    main()
