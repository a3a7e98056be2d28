#!/usr/bin/env python
"""Benchmark of the leapfrog hot path (BASELINE.json metric: 2D stencil Gpoint-updates/s and HBM
GB/s vs the B200 peak, at 1/2/4/8 GPUs).

Workload: config 4's weak-scaling unit (R22) — a 32768 × 4096-row δ-line slab per
GPU (global grid 32768 × 4096·N, dx = dy = 0.0025, ε = 0.05, dt = 4e−4), dense uniform [−1, 1]
data (SURVEY §8(d) data-independence guard), fp64 by default.  One "step" = one pass of the
hot path over the slab: the leapfrog stencil (S3), the NCCL ghost-row exchange at N > 1 (S4),
and the discrete-energy reduction every `--energy-every` steps (S5).  By default the stencil is
temporally blocked (K = 10 levels per HBM pass in both precisions by default; a stepping call's
remainder of r < K levels is one pass of depth r; K-deep ghost rows on slabs); `--tblock 1` times
the one-level-per-pass kernel.  Inputs (2 × 1.07 GB per
GPU in fp64) exceed the 126 MB L2, so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype f64|f32] [--impl tsw|reference]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2D stencil Gpoint-updates/s & HBM GB/s vs 8 TB/s peak, at 1/2/4/8 B200"
UNIT = "Gpt/s"
ESZ = {"f64": 8, "f32": 4}
TB_DEFAULT = {"f64": 10, "f32": 10}   # levels per HBM pass (round-2 sweep on B200: 10 ≥ 8 per pass, and a
                                      # 20- or 100-level call needs no shallower remainder pass)


def words_per_update(steps: int, cadence: int, K: int) -> float:
    """Algorithmic HBM words per point-update of the timed loop: a one-level step
    moves 3 words per node (read u^n, u^{n-1}; write u^{n+1}), a temporally blocked pass of any
    depth 4 (read u^n, u^{n-1}; write u^{n+K}, u^{n+K-1}).  A stepping call of q·K + r levels runs
    q passes of depth K and, for r >= 2, one pass of depth r (r = 1: one level)."""
    words = levels = 0
    done = 0
    while done < steps:
        k = min(cadence, steps - done) if cadence > 0 else steps - done
        if K <= 1:
            words += 3 * k
        else:
            q, r = divmod(k, K)
            words += 4 * (q + (1 if r >= 2 else 0)) + (3 if r == 1 else 0)
        levels += k
        done += k
    return words / levels


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _sm_max_mhz() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["sm_max_mhz"])
    except Exception:
        return 1965.0   # B200 maximum SM clock


SM_MAX_MHZ = _sm_max_mhz()


def alu_peak(dtype: str) -> float:
    """Derived non-FMA arithmetic roof in TFLOP/s: 64 fp64 / 128 fp32 lanes per clock per
    SM, 148 SMs, maximum SM clock — the fallback when the probe is unavailable."""
    return (64.0 if dtype == "f64" else 128.0) * 148 * SM_MAX_MHZ * 1e6 / 1e12


def alu_roof(dtype: str, device: int):
    """(TOP/s, source) of the ALU roof: measured on this GPU by tsw_alu_probe (independent
    non-contracted add/multiply chains on every SM, best of 3), else the derived figure."""
    try:
        from paper_2005_11931_b200 import tsw
        v = tsw.tsw_alu_probe(device, tsw.TSW_F64 if dtype == "f64" else tsw.TSW_F32) / 1e12
        return v, ("measured (tsw_alu_probe: %s add/mul chains on all SMs, best of 3; derived nominal %.2f)"
                   % (dtype, alu_peak(dtype)))
    except Exception as e:  # noqa: BLE001 — reported in the line
        return alu_peak(dtype), "derived (probe failed: %s): %d lanes/clk/SM x 148 SMs x %.0f MHz" % (
            e, 64 if dtype == "f64" else 128, SM_MAX_MHZ)


def ncu_traffic(dtype: str, workload: str, tblock: int = 1, kernel: str = ""):
    """dram bytes per launch of the dominant kernel from the committed ncu summaries, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get(f"{dtype}_{kernel}" if kernel else (dtype if tblock == 1 else f"{dtype}_tb{tblock}"))
        if e and e.get("workload") == workload:
            return float(e["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled in the background (the recipe's clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.samples = []
        self.proc = None
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))

    def wait_ready(self, timeout: float = 5.0):
        t0 = time.time()
        while self.proc and not self.samples and time.time() - t0 < timeout:
            time.sleep(0.05)

    def mark(self, start: bool):
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        win = [s for t, s in self.samples if self.t0 is not None and self.t0 - 0.06 <= t <= (self.t1 or t) + 0.06]
        if not win and self.samples:
            # the timed region was shorter than the sampling period: nearest sample
            mid = 0.5 * ((self.t0 or 0) + (self.t1 or 0))
            win = [min(self.samples, key=lambda ts: abs(ts[0] - mid))[1]]
        sm = [float(s[0]) for s in win if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in win if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in win for k in range(4) if len(s) > 4 + k and s[4 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(win)}


def cpu_baseline(cfg, dtype: str, budget_s: float = 15.0, rows: int = 1024):
    """The oracle as it stands, on this host's cores, over a bounded sample of the same workload:
    `rows` interior rows × the full 32768-wide row, dense data, the same δ-line faces."""
    import oracle
    threads = host_cores()
    oracle.set_threads(threads)
    npdt = np.float64 if dtype == "f64" else np.float32
    j0 = cfg.ny // 2 - rows // 2
    wny = rows + 2
    _, _, c1, c2 = oracle.member_coefficients(cfg, 0, npdt, 0, j0, cfg.nx, wny)
    from paper_2005_11931_b200 import inputs
    u = inputs.uniform_dense_rows(cfg.nx, cfg.ny, j0, wny).astype(npdt)
    v = oracle.startup(2, c1, c2, u, None, cfg.dt)
    # doubling chunks of leapfrog steps until the budget is spent (each call also copies the slab)
    oracle.leapfrog(2, c1, c2, v, u, 1)
    steps, el, k = 0, 0.0, 8
    while el < budget_s and steps < 20000:
        t = time.perf_counter()
        v, u = oracle.leapfrog(2, c1, c2, v, u, k)
        el += time.perf_counter() - t
        steps += k
        k *= 2
    upd = rows * (cfg.nx - 2) * steps
    cores = int(oracle.max_threads())
    # the same sample on one core (1-core and all-core rates), ≈ budget / 4
    oracle.set_threads(1)
    s1, e1, k = 0, 0.0, 2
    while e1 < budget_s / 4 and s1 < 2000:
        t = time.perf_counter()
        v, u = oracle.leapfrog(2, c1, c2, v, u, k)
        e1 += time.perf_counter() - t
        s1 += k
        k *= 2
    oracle.set_threads(threads)
    return {"value": upd / el / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "value_1core": rows * (cfg.nx - 2) * s1 / e1 / 1e9,
            "sample": f"{rows} rows x {cfg.nx} cols of the per-GPU slab, {steps} leapfrog steps, {dtype}, "
                      f"OpenMP over rows, {el:.1f} s (1 core: {s1} steps, {e1:.1f} s)"}


def run_reference(args, cfg, rank: int, world: int):
    """--impl reference: the oracle (this tier's reference arm) on the host cores, rank 0 only."""
    if rank != 0:
        return 0
    import oracle
    from paper_2005_11931_b200 import inputs
    threads = host_cores()
    oracle.set_threads(threads)
    npdt = np.float64 if args.dtype == "f64" else np.float32
    rows = args.ref_rows
    j0 = cfg.ny // 2 - rows // 2
    _, _, c1, c2 = oracle.member_coefficients(cfg, 0, npdt, 0, j0, cfg.nx, rows + 2)
    u = inputs.uniform_dense_rows(cfg.nx, cfg.ny, j0, rows + 2).astype(npdt)
    v = oracle.startup(2, c1, c2, u, None, cfg.dt)
    if args.warmup:
        v, u = oracle.leapfrog(2, c1, c2, v, u, args.warmup)
    t = time.perf_counter()
    oracle.leapfrog(2, c1, c2, v, u, args.steps)
    el = time.perf_counter() - t
    upd = rows * (cfg.nx - 2) * args.steps
    val = upd / el / 1e9
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": args.dtype, "impl": "reference",
            "data": "synthetic (dense uniform[-1,1], seed 0)",
            "config": {"workload": workload_name(cfg, world), "sample_rows": rows, "nx": cfg.nx},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": int(oracle.max_threads()), "kind": "oracle",
                             "sample": f"{rows} rows x {cfg.nx} cols per step of the per-GPU slab"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --- Table 1 workload: the paper's implicit method -----------------------

PAPER_T1_GPU_S = 62.76   # PAPER.md Table 1, RTX 2080 Ti, 4096², 100 steps — context only
T1_N, T1_DT, T1_EPS = 4096, 0.05, 0.8


def table1_scenario():
    from paper_2005_11931_b200 import inputs
    return inputs.paper_2d(dx=100.0 / (T1_N - 1))     # [0,100]² as N² nodes, H = h_0(x), Gaussian u0


def table1_oracle_coeffs(sc, npdt):
    """Prescaled faces for the oracle: the profile depends on x only, so one row is built and tiled."""
    import oracle
    prof = oracle.Profile(sc.seg_value, sc.seg_break, sc.sing_loc, sc.sing_amp, sc.sing_order, sc.isotropic)
    h1r, h2r = oracle.build_faces_profile(2, prof, T1_EPS, sc.nx, sc.ny, sc.dx, j0=0, wny=2)
    c1 = oracle.prescale(np.ascontiguousarray(np.broadcast_to(h1r[:1], (sc.ny, sc.nx - 1))), T1_DT, sc.dx, npdt)
    c2 = oracle.prescale(np.ascontiguousarray(np.broadcast_to(h2r[:1], (sc.ny - 1, sc.nx))), T1_DT, sc.dx, npdt)
    return c1, c2


def table1_oracle_rate(dtype: str, budget_s: float, max_steps: int):
    """Implicit levels of the oracle (Thomas line solves, OpenMP over lines) on the full grid."""
    import oracle
    threads = host_cores()
    oracle.set_threads(threads)
    npdt = np.float64 if dtype == "f64" else np.float32
    sc = table1_scenario()
    c1, c2 = table1_oracle_coeffs(sc, npdt)
    u0 = sc.initial().astype(npdt)
    steps, el = 0, 0.0
    while el < budget_s and steps < max_steps:
        t = time.perf_counter()
        oracle.implicit_run(2, c1, c2, u0, None, T1_DT, 1)
        el += time.perf_counter() - t
        steps += 1
    upd = (sc.nx - 2) * (sc.ny - 2) * steps
    return upd / el / 1e9, int(oracle.max_threads()), steps, el


def run_table1(args, rank: int, world: int, local: int):
    """--workload table1: one step = one implicit level (x-line solves, y-line solves, three-level
    update) over the 4096² grid; N GPUs run N replicas (the implicit path is single-rank)."""
    wl = f"table1_implicit_{T1_N}x{T1_N}_per_gpu"
    if args.impl == "reference":
        if rank != 0:
            return 0
        val, cores, steps, el = table1_oracle_rate(args.dtype, 1e9, max(1, args.steps))
        line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * el / steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "impl": "reference",
                "data": "synthetic (paper Gaussian u0, P:1156; H = h_0(x), eps 0.8)",
                "config": {"workload": wl, "scheme": "implicit (oracle, Thomas)", "dt": T1_DT},
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                                 "sample": f"{steps} implicit levels on the full {T1_N}^2 grid"},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist
    from paper_2005_11931_b200 import parallel, tsw
    torch.cuda.set_device(local)
    if world > 1:
        parallel.init_process_group("nccl")
    dev = torch.device("cuda", local)
    sc = table1_scenario()
    esz = ESZ[args.dtype]
    npdt = np.float64 if args.dtype == "f64" else np.float32

    def make(dtype):
        stream = torch.cuda.Stream(device=dev)
        s = tsw.Solver(2, sc.nx, sc.ny, sc.dx, sc.dx, 1, dtype, device=local, stream=stream.cuda_stream)
        s.set_coeff_profile(sc.seg_value, sc.seg_break, [T1_EPS], isotropic=True)
        s.set_option(tsw.TSW_OPT_SCHEME, 1)
        return s, stream

    s, stream = make(args.dtype)
    u0_host = torch.from_numpy(sc.initial().astype(npdt)[None]).pin_memory()
    u0_dev = u0_host.to(dev)
    torch.cuda.synchronize()
    s.set_initial(u0_dev, None, T1_DT)
    clocks = ClockSampler(local)
    s.step(max(20, 3 * args.warmup))            # untimed spin-up (clocks ramp), then warm-up
    s.step(args.warmup)
    clocks.wait_ready()
    s.set_option(tsw.TSW_OPT_TIME_KERNELS, 1)
    l0 = s.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark(True)
    ev0.record(stream)
    s.step(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(False)
    ms = ev0.elapsed_time(ev1)
    launches = s.launches() - l0
    kms, kl, kupd = s.kernel_stats()
    s.set_option(tsw.TSW_OPT_TIME_KERNELS, 0)
    kavg = kms / max(kl, 1)
    if world > 1:
        t = torch.tensor([ms, kavg], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kavg = float(t[0]), float(t[1])
    clk = clocks.stop()
    upd = (sc.nx - 2) * (sc.ny - 2) * args.steps * world
    value = upd / (ms * 1e-3) / 1e9
    # e2e: H2D of u0 (pinned), K levels, D2H of u^K
    out_host = torch.empty((1, sc.ny, sc.nx), dtype=u0_host.dtype).pin_memory()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.set_initial(u0_host.numpy(), None, T1_DT)
    s.step(args.steps)
    s.read(0, out_host.numpy())
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t[0])
    s.close()
    if rank == 0:
        peak, peak_src = measured_peak()
        # the timed kernel of the library's automatic solver choice (TSW_OPT_IMPLICIT_SOLVER = 0)
        ykern = "imp_yfin" if (args.dtype == "f64" and (sc.nx - 2) * (sc.ny - 2) >= (8 << 20)) else "imp_yc"
        per_launch = kupd / max(kl, 1)
        achieved = per_launch * 3 * esz / (kavg * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (paper Gaussian u0 50exp(-((x-40)^2+(y-50)^2)/8), P:1156; H = h_0(x), eps 0.8)",
            "config": {"workload": wl, "scheme": "implicit factorised CN (R26/R27), scan line solvers (R28, automatic y-solve variant)",
                       "nx": sc.nx, "ny": sc.ny, "dx": sc.dx, "dt": T1_DT,
                       "parallelism": f"{world} independent replicas" if world > 1 else "single GPU",
                       "l2": "fields 2 x %.0f MB + scratch exceed L2, no flush" % (sc.nx * sc.ny * esz / 1e6),
                       "paper_table1_gpu_s_100_steps": PAPER_T1_GPU_S,
                       "this_run_s_100_steps": ms / args.steps * 100 / 1e3},
            "hbm_gbs_effective": value * 5 * esz,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(args.dtype, wl, kernel=ykern),
                         "kernel": f"k_{ykern} (y-line closed-form solve + three-level update)",
                         "algorithmic_bytes_per_update": 3 * esz, "peak_source": peak_src, "kernel_avg_ms": kavg,
                         "level_algorithmic_bytes_per_node": 5 * esz,
                         "level_frac": value * 5 * esz / peak},
            "gpu_launches": launches, "clocks": clk,
            "e2e": {"value": upd / el / 1e9, "unit": UNIT, "h2d_bytes_per_step": u0_host.numel() * esz / args.steps,
                    "d2h_bytes_per_step": out_host.numel() * esz / args.steps},
        }
        if world == 1 and not args.no_cpu_baseline:
            v, cores, st, tt = table1_oracle_rate(args.dtype, 15.0, 200)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": f"{st} implicit levels on the full {T1_N}^2 grid ({tt:.1f} s)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def workload_name(cfg, world: int) -> str:
    if cfg.name.startswith("config4_strong"):
        return f"config4_strong_{cfg.nx}x{cfg.ny}_over_{world}_gpus"
    if cfg.batch > 1:
        return f"config5_eps_family_{cfg.batch}x{cfg.nx}x{cfg.ny // world}_per_gpu"
    if cfg.name.startswith("config3"):
        return f"config3_delta_line_{cfg.nx}x{cfg.ny // world}_per_gpu"
    return f"config4_weak_unit_delta_line_{cfg.nx}x{cfg.ny // world}_per_gpu"


def relaunch(n: int) -> int:
    """`bench.py --gpus N` started as one process: re-run the same command line under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous, a free port), as the driver's
    multi-GPU launch does; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", str(max(1, host_cores() // n))))
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64")
    ap.add_argument("--impl", choices=["tsw", "reference"], default="tsw")
    ap.add_argument("--rows-per-gpu", type=int, default=4096)
    ap.add_argument("--nx", type=int, default=32768)
    ap.add_argument("--energy-every", type=int, default=100)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-also", action="store_true", help="skip the second-precision line item")
    ap.add_argument("--ref-rows", type=int, default=64)
    ap.add_argument("--rows-per-item", type=int, default=0)
    ap.add_argument("--workload", choices=["config4", "config5", "config3", "table1"], default="config4",
                    help="config4: the weak-scaling unit (default, the BASELINE metric's scaling "
                         "workload); config5: 65-member eps family x 2048^2; config3: 4096^2 delta line; "
                         "table1: the paper's implicit method on its Table 1 set-up (4096^2, dt 0.05)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: 32768 x rows-per-gpu per GPU (default); strong: the 32768^2 grid split over the GPUs (R22)")
    ap.add_argument("--halo", choices=["peer", "nccl"], default="nccl",
                    help="ghost rows of the row slabs at N > 1: NCCL send/recv of the K boundary rows on the aux "
                         "stream, overlapped with the interior rows (default, the north_star path) or peer stores "
                         "fused into the stencil over NVLink (CUDA IPC)")
    ap.add_argument("--tblock", type=int, default=0,
                    help="levels per HBM pass of the temporally blocked stencil (1 = per-step TMA kernel; "
                         "0 = per dtype: 4 for f64, 8 for f32 — the sweep optimum, tools/sweep.py)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    from paper_2005_11931_b200 import inputs, parallel
    rank, world, local = parallel.env_rank()
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
    if args.impl != "reference":
        import torch
        if torch.cuda.device_count() < min(world, local + 1) or not torch.cuda.is_available():
            sys.stderr.write(f"bench.py: rank {rank} needs GPU {local}, {torch.cuda.device_count()} visible\n")
            return 2
    if args.workload == "table1":
        return run_table1(args, rank, world, local)
    if args.workload == "config5":
        cfg = inputs.config(5, ny=2048 * world)
    elif args.workload == "config3":
        cfg = inputs.config(3, ny=4096 * world)
    else:
        if args.scaling == "strong":   # R22: the fixed 32768² grid split over the ranks
            cfg = inputs.config(4, nx=args.nx, ny=args.nx, name=f"config4_strong_{args.nx}x{args.nx}")
        else:
            cfg = inputs.weak_unit(world, rows_per_rank=args.rows_per_gpu, nx=args.nx)

    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    # S5 in every timed region: the energy cadence is capped at the step count (an energy call
    # at the end of the timed steps even for --steps < --energy-every)
    cadence = min(args.energy_every, args.steps) if args.energy_every > 0 else 0

    import torch
    import torch.distributed as dist
    from paper_2005_11931_b200 import tsw
    torch.cuda.set_device(local)
    if world > 1:
        parallel.init_process_group("nccl")
    dev = torch.device("cuda", local)

    halo_used, halo_note = ["nccl"], []

    def run(dtype: str, full: bool, tblock: int):
        npdt = np.float64 if dtype == "f64" else np.float32
        stream = torch.cuda.Stream(device=dev)
        s = tsw.Solver.from_config(cfg, dtype, rank=rank, nranks=world, device=local, stream=stream.cuda_stream)
        if args.rows_per_item:
            s.set_option(tsw.TSW_OPT_ROWS_PER_ITEM, args.rows_per_item)
        if tblock > 1:
            s.set_option(tsw.TSW_OPT_TBLOCK, tblock)
        parallel.nccl_bootstrap(s)            # the communicator serves the reductions (energy)
        if world > 1 and args.halo == "peer":
            # ghost rows by peer stores from the stencil itself (fused halo push over NVLink);
            # every rank must agree, so a failure anywhere falls back to NCCL halos everywhere
            ok = True
            try:
                parallel.peer_bootstrap(s)
            except Exception as e:  # noqa: BLE001 — reported in the JSON line
                ok = False
                halo_note.append(f"peer halos unavailable on rank {rank}: {e}")
            flag = torch.tensor([1.0 if ok else 0.0], device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if flag.item() < 1.0:
                s.set_option(tsw.TSW_OPT_HALO, 0)
                halo_used[0] = "nccl"
            else:
                halo_used[0] = "peer"
        r0, r1 = parallel.slab(cfg.ny, rank, world)
        u0_host = torch.from_numpy(inputs.uniform_dense_rows(cfg.nx, cfg.ny, r0, r1 - r0).astype(npdt)).pin_memory()
        # (config 5: every member starts from the same field — TSW_INIT_SHARED)
        u0_dev = u0_host.to(dev)
        torch.cuda.synchronize()
        s.set_initial(u0_dev, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
        # untimed spin-up (clocks ramp) then the W warm-up steps; the clock sampler starts first
        # and must have delivered a sample before the timed region begins
        clocks = ClockSampler(local) if full else None
        s.step(max(50, 3 * args.warmup))
        s.step(args.warmup)
        s.energy()
        if clocks:
            clocks.wait_ready()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.set_option(tsw.TSW_OPT_TIME_KERNELS, 1)
        l0 = s.launches()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if clocks:
            clocks.mark(True)
        ev0.record(stream)
        done = 0
        while done < args.steps:
            k = min(cadence, args.steps - done) if cadence > 0 else args.steps - done
            s.step(k)
            done += k
            if cadence > 0 and done % cadence == 0:
                s.energy()
        ev1.record(stream)
        torch.cuda.synchronize()
        if clocks:
            clocks.mark(False)
        if world > 1:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        launches = s.launches() - l0
        kms, klaunch, kupd = s.kernel_stats()
        lms, llev, lupd = s.kernel_launches()
        s.set_option(tsw.TSW_OPT_TIME_KERNELS, 0)
        # the dominant kernel: the launches of the full depth (K-level passes; a call's shallower
        # remainder pass is reported separately, not averaged in)
        full_k = int(llev.max()) if len(llev) else 1
        sel = llev == full_k
        pass_ms = float(lms[sel].mean()) if sel.any() else kms / max(klaunch, 1)
        pass_upd = float(lupd[sel].mean()) if sel.any() else kupd / max(klaunch, 1)
        if world > 1:
            t = torch.tensor([pass_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pass_ms = float(t[0])
        if world > 1:
            t = torch.tensor([ms, kms / max(klaunch, 1)], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, kavg = float(t[0]), float(t[1])
        else:
            kavg = kms / max(klaunch, 1)
        updates = (cfg.nx - 2) * (cfg.ny - 2) * cfg.batch * args.steps
        res = {"ms": ms, "value": updates / (ms * 1e-3) / 1e9, "launches": launches, "kernel_avg_ms": kavg,
               "kernel_updates_per_launch": kupd / max(klaunch, 1), "clocks": clocks.stop() if clocks else None,
               "pass_levels": full_k, "pass_ms": pass_ms, "pass_updates": pass_upd,
               "pass_count": int(sel.sum()), "timed_launch_levels": [int(x) for x in llev]}
        if full and not args.no_e2e:
            # e2e through the public API with host buffers: H2D of u0 (pinned), K steps (+ energy),
            # D2H of u^K — all inside the timed region.
            out_host = torch.empty((cfg.batch, r1 - r0, cfg.nx), dtype=u0_host.dtype).pin_memory()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s.set_initial(u0_host.numpy(), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
            done = 0
            while done < args.steps:
                k = min(cadence, args.steps - done) if cadence > 0 else args.steps - done
                s.step(k)
                done += k
                if cadence > 0 and done % cadence == 0:
                    s.energy()
            s.read(0, out_host.numpy())
            el = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([el], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                el = float(t[0])
            nb = u0_host.numel() * u0_host.element_size()
            nbo = out_host.numel() * out_host.element_size()
            res["e2e"] = {"value": updates / el / 1e9, "unit": UNIT, "h2d_bytes_per_step": nb / args.steps,
                          "d2h_bytes_per_step": nbo / args.steps}
        if world > 1:
            dist.barrier()   # every rank's streams are done (peer halos write into neighbours' buffers)
        s.close()
        del u0_dev
        torch.cuda.empty_cache()
        return res

    # slabs exchange K ghost rows of both levels every K levels
    tblock = args.tblock or TB_DEFAULT[args.dtype]
    roofs = {dt: alu_roof(dt, local) for dt in ("f64", "f32")}
    main_res = run(args.dtype, True, tblock)
    other = "f32" if args.dtype == "f64" else "f64"
    tblock_other = args.tblock or TB_DEFAULT[other]
    also = None if args.no_also else run(other, False, tblock_other)
    per_step = None
    if tblock > 1 and not args.no_also:
        per_step = run(args.dtype, False, 1)  # the one-level-per-pass kernel on the same workload

    if rank == 0:
        peak, peak_src = measured_peak()
        esz = ESZ[args.dtype]
        # algorithmic bytes per point-update: 3 words per step; with temporal
        # blocking, (2 reads + 2 writes) per pass (words_per_update)
        words = words_per_update(args.steps, cadence, tblock)
        # the dominant kernel: the full-depth launches (K-level passes; a call's shallower remainder
        # pass is not averaged in), live CUDA-event times on the ctx stream
        kp = main_res["pass_levels"]
        upd_s = main_res["pass_updates"] / (main_res["pass_ms"] * 1e-3)
        words_pass = 4.0 / kp if kp > 1 else 3.0           # algorithmic words per update in one launch
        achieved = upd_s * words_pass * esz / 1e9
        wl = workload_name(cfg, world)
        traffic = ncu_traffic(args.dtype, wl, tblock)
        hbm_frac = achieved / peak
        # ALU roof: the measured non-contracted add/multiply rate of this GPU (tsw_alu_probe) against
        # the 14 operations per update of the canonical tree (algorithmic count)
        fp_peak, fp_src = roofs[args.dtype]
        alu_ach = upd_s * 14 / 1e12
        alu_frac = alu_ach / fp_peak
        hbm_obj = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": hbm_frac,
                   "traffic": traffic, "algorithmic_bytes_per_update": words * esz, "peak_source": peak_src}
        alu_obj = {"bound": "alu", "achieved": alu_ach, "peak": fp_peak, "unit": "TFLOP/s", "frac": alu_frac,
                   "traffic": traffic, "ops_per_update": 14, "peak_source": fp_src}
        # the binding roof is the one the kernel is closer to; the other is reported beside it
        roof, other_view = (alu_obj, hbm_obj) if alu_frac > hbm_frac else (hbm_obj, alu_obj)
        line = {
            "metric": METRIC, "value": main_res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main_res["ms"] / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (dense uniform[-1,1] u0, u1 = 0, seed 0; delta-line h_eps, eps = 0.05)",
            "config": {"workload": wl, "nx": cfg.nx, "ny_global": cfg.ny, "rows_per_gpu": cfg.ny // world,
                       "batch": cfg.batch, "dx": cfg.dx, "dt": cfg.dt,
                       "eps": cfg.eps[0] if cfg.batch == 1 else [min(cfg.eps), max(cfg.eps)],
                       "energy_every": cadence,
                       "temporal_blocking": tblock,
                       "parallelism": (f"row-slab x{world} (" + ("peer-store ghost rows fused into the stencil, NVLink"
                                                                  if halo_used[0] == "peer" else "NCCL ghost rows") + ")")
                       if world > 1 else "single GPU",
                       "halo_notes": halo_note or None,
                       "l2": "inputs exceed L2 (2 levels x %.2f GB per GPU), no flush" %
                             ((cfg.nx * (cfg.ny // world) * esz * cfg.batch) / 1e9)},
            "hbm_gbs_effective": main_res["value"] * words * esz,
            "roofline": {**roof,
                         "kernel": ("k_step2d_tma (S3 leapfrog, one level per pass)" if tblock == 1 else
                                    f"k_step2d_tb (S3 leapfrog, K={tblock} levels per HBM pass)"),
                         "kernel_avg_ms": main_res["pass_ms"], "kernel_levels": kp,
                         "kernel_launches_timed": main_res["pass_count"],
                         "timed_launch_levels": main_res["timed_launch_levels"],
                         "all_launches_avg_ms": main_res["kernel_avg_ms"],
                         "per_step_roofline_gpts": peak / (3 * esz),
                         ("alu_view" if roof is hbm_obj else "hbm_view"): other_view},
            "gpu_launches": main_res["launches"],
            "clocks": main_res["clocks"],
            "context": {"paper_table1": "implicit cyclic-reduction scheme (a different algorithm), 4096^2, 100 steps: "
                                        "62.76 s on an NVIDIA GeForce RTX 2080 Ti vs 280.54 s serial on an Intel Core "
                                        "i7-9800X (speedup 4.47, P:1168-1183); this repo's implicit path: "
                                        "bench.py --workload table1",
                        "note": "context only, not a target (BASELINE.md section 2)"},
        }
        if "e2e" in main_res:
            line["e2e"] = main_res["e2e"]
        if also:
            e2 = ESZ[other]
            words2 = words_per_update(args.steps, cadence, tblock_other)
            kp2 = also["pass_levels"]
            upd2 = also["pass_updates"] / (also["pass_ms"] * 1e-3)
            ach2 = upd2 * (4.0 / kp2 if kp2 > 1 else 3.0) * e2 / 1e9
            line["also"] = {"dtype": other, "value": also["value"], "unit": UNIT, "temporal_blocking": tblock_other,
                            "ms_per_step": also["ms"] / args.steps, "roofline_frac": ach2 / peak, "achieved_gbs": ach2,
                            "alu_frac": upd2 * 14 / 1e12 / roofs[other][0], "kernel_avg_ms": also["pass_ms"],
                            "alu_peak": roofs[other][0]}
        if per_step:
            ach1 = per_step["kernel_updates_per_launch"] * 3 * esz / (per_step["kernel_avg_ms"] * 1e-3) / 1e9
            line["per_step_kernel"] = {"kernel": "k_step2d_tma", "value": per_step["value"], "unit": UNIT,
                                       "achieved_gbs": ach1, "roofline_frac": ach1 / peak,
                                       "traffic": ncu_traffic(args.dtype, wl, 1)}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, args.dtype)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
