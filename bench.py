#!/usr/bin/env python
"""Benchmark of the full-order implicit time step (BASELINE.json north_star).

Workload (BASELINE configs[2], "large", the largest single-GPU config): 128x128x256
voxel half cell (6.5 M DOF), 3C constant-current charge, dt = 0.25 s, plating/stripping
on, fp64, at the config's stated tolerances: Newton relative tolerance 1e-8, Krylov
relative tolerance 1e-10 on every Newton system.  One bench step = one accepted
implicit-Euler step (Newton + preconditioned Krylov + plated-inventory update) through
the C ABI (``hc_step``) on device-resident state.  ``value`` = implicit steps/s over all
ranks (each rank steps its own cell: replicas, no data-path collective).  ``e2e`` = the
same K steps through ``hc_step_host`` with pinned host state buffers (H2D + D2H inside
the timed region, L2 flushed before each step like ``value``).  The residual and J v
kernels are timed separately (CUDA events, L2 flushed before every launch) for the
GDOF/s figures and the roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--impl reference`` times the CPU oracle port of the reference algorithm
(oracle/fvm_oracle.py, SuperLU-based Newton like fvm/newton.py:75-77) on a
bounded sample of the same workload with all host cores (rank 0 only).
"""

from __future__ import annotations

import argparse
import ctypes
import dataclasses
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "implicit time steps/s and residual+J*v GDOF/s; % of B200 HBM roofline"
FALLBACK_HBM_GBS = 6650.0
L2_FLUSH_BYTES = 256 << 20
# Krylov tolerance of Newton iteration k: max(linear_rtol, safety * tol / |F_k|); the
# headline uses 0 (BASELINE's Krylov rtol 1e-10 on every system); the inexact-Newton
# figure (0.3, curve parity in tests/test_gpu_configs.py) is reported beside it
LINEAR_SAFETY = float(os.environ.get("HC_BENCH_LINEAR_SAFETY", "0.0"))
INEXACT_SAFETY = 0.3


def solver_config(P, config: str, rs, safety: float):
    """SolverConfig of a BASELINE run: configs[2] states Newton 1e-8 / Krylov 1e-10; the
    other configs use the reference's SolverConfig defaults (newton.py:20-34)."""
    kw = dict(newton_rtol=1e-8, linear_rtol=1e-10) if config == "large" else {}
    return P.SolverConfig(dt_init=min(0.05, rs.dt), dt_max=rs.dt, linear_safety=safety, **kw)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cell_for(config: str, rank: int):
    from paper_1704_04139_b200.configs import CONFIGS
    rs = CONFIGS[config]
    spec = dataclasses.replace(rs.cell, seed=rs.cell.seed + 1000 * rank) if rank else rs.cell
    return rs, spec


def drive_mu(labels, voxel_um, c_rate, params):
    """Charge current density (A/m^2, negative = lithiation) for a C-rate of the graphite."""
    h = voxel_um * 1e-6
    vol_gr = float(np.count_nonzero(labels == 1)) * h ** 3
    area = labels.shape[1] * labels.shape[2] * h * h
    return -c_rate * params.c_gr_max * params.constants.F * vol_gr / 3600.0 / area


def committed_traffic(config: str, kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/traffic.json, written from the .ncu-rep of the same bench command)."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d.get(config, {}).get(kernel)
    except Exception:
        return None


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU baseline
def _oracle_column_step(args):
    """One implicit step of the CPU oracle on a w x w column of the workload cell."""
    config, w, seed = args
    from oracle import fvm_oracle as O
    from paper_1704_04139_b200.configs import CONFIGS
    from paper_1704_04139_b200.microgen import generate_cell
    from paper_1704_04139_b200.errors import GeometryError
    rs = CONFIGS[config]
    for attempt in range(20):   # a thin column can miss the collector; take the next seed
        try:
            grid = generate_cell(dataclasses.replace(rs.cell, nx=w, ny=w, seed=seed + 100000 * attempt))
            break
        except GeometryError:
            continue
    p = O.Params(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
    op = O.OracleOperator(grid.labels, grid.voxel_size, p)
    h = grid.voxel_size * 1e-6
    mu = -rs.c_rate * p.c_gr_max * p.F * np.count_nonzero(grid.labels == 1) * h ** 3 / 3600 / (w * w * h * h)
    x, npl = O.initial_fields(op)
    x = O.solve_initial_potential(op, x, npl, mu)
    t0 = time.perf_counter()
    O.step(op, x, npl, rs.dt, mu)
    return time.perf_counter() - t0


def cpu_sample(config: str, rounds: int, warmup: int = 0):
    """Parallel oracle column steps on all host cores; returns per-round cell-steps/s."""
    import multiprocessing as mp
    from paper_1704_04139_b200.configs import CONFIGS
    rs = CONFIGS[config]
    w = 8 if config == "large" else 16
    frac = (w * w) / (rs.cell.nx * rs.cell.ny)
    cores = max(1, min(os.cpu_count() or 1, 16))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    vals = []
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        for r in range(warmup + rounds):
            t0 = time.perf_counter()
            pool.map(_oracle_column_step, [(config, w, 7000 + 97 * r + k) for k in range(cores)])
            wall = time.perf_counter() - t0
            if r >= warmup:
                vals.append(cores * frac / wall)
    sample = (f"{cores} concurrent implicit steps of the CPU oracle (SuperLU Newton, fvm/newton.py:75-77) "
              f"on {w}x{w}x{rs.cell.nz} columns of the {config} cell ({frac:.5f} of its voxels each); "
              "the cell's rate is EXTRAPOLATED linearly by voxel count (favourable to the CPU: "
              "sparse LU cost grows superlinearly)")
    return vals, cores, sample


# ------------------------------------------------------------------ GPU arm
def kernel_roofline(op, grid, params, x, npl, beta, dt, config):
    """CUDA-event times of the residual and J v kernels (L2 read-flushed before every
    launch) and the J v roofline: algorithmic bytes / launch time vs the measured peak."""
    import ctypes
    from paper_1704_04139_b200 import _dev, _native
    L = _native.lib()
    ms = (ctypes.c_double * 5)()
    _native.check(L.hc_time_kernels(op.native.handle, _dev.ptr(x), _dev.ptr(npl), beta, 1.0 / dt, 20,
                                    L2_FLUSH_BYTES, ms, _dev.stream()))
    info = op.native.info
    nvox = int(info.n_vox)
    n_el = int(np.count_nonzero(grid.labels == 0))
    n_c = int(np.count_nonzero(np.isin(grid.labels, (0, 1))))
    n_if = int(info.n_bv + info.n_ce + info.n_strip)
    res_ms, jv_ms = ms[0] + ms[1], ms[2] + ms[3]
    # labels + v (c, phi) + out + gX/c on electrolyte voxels + 3 linearized coefficients per interface face
    jv_bytes = nvox * (1 + 16 + 16) + n_el * 8 + n_if * 24
    res_bytes = nvox * (1 + 16 + 16) + n_c * 8          # labels + x + out + c_prev
    peak, peak_kind = measured_peaks()
    achieved = jv_bytes / (ms[2] * 1e-3) / 1e9
    copy_gbs = nvox * 32 / (ms[4] * 1e-3) / 1e9          # same-size streaming copy, same timing
    traffic = committed_traffic(config, "k_fine_tma<0, 0, 1>")
    return {
        "res_ms": res_ms, "jv_ms": jv_ms,
        "kernel_ms": {"residual_stencil": ms[0], "residual_iface": ms[1],
                      "jvp_stencil": ms[2], "jvp_iface": ms[3]},
        "roofline": {"kernel": "k_fine_tma<SM_FULL> (J v: TMA tiles, fused interface slots)",
                     "bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "bytes_per_launch": jv_bytes,
                     "bytes_per_voxel": "label 1 + v 16 + out 16 (+ gX/c 8 per electrolyte voxel, "
                                        "+ 24 per interface face)",
                     "grid": f"{grid.labels.shape[2]}x{grid.labels.shape[1]}x{grid.labels.shape[0]}",
                     "same_size_stream_copy_gbs": copy_gbs,
                     "frac_of_stream_copy": achieved / copy_gbs,
                     "residual": {"kernel": "k_fine_tma<SM_RES> + k_residual_islot",
                                  "achieved": res_bytes / (res_ms * 1e-3) / 1e9,
                                  "frac": res_bytes / (res_ms * 1e-3) / 1e9 / peak,
                                  "bytes_per_launch": res_bytes}},
    }


def roofline_at_scale():
    """J v / residual kernel roofline on the large config's grid (128x128x256) at its
    initial state: the same kernels with an HBM-resident working set."""
    import paper_1704_04139_b200 as P
    from paper_1704_04139_b200 import _dev
    from paper_1704_04139_b200.microgen import generate_cell
    from paper_1704_04139_b200.state import initial_fields
    rs, spec = cell_for("large", 0)
    grid = generate_cell(spec)
    params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
    dof = P.build_dofmap(grid)
    op = P.SystemOperator(dof, params)
    st = initial_fields(dof, params)
    x = _dev.to_dev(st.x)
    npl = _dev.to_dev(st.n_pl if st.n_pl.size else np.zeros(1))
    beta = rs.dt * op.face_area / params.constants.F
    kt = kernel_roofline(op, grid, params, x, npl, beta, rs.dt, "large")
    out = dict(kt["roofline"])
    out["kernel_ms"] = kt["kernel_ms"]
    out["state"] = "initial fields of the large config"
    del op
    return out


def workload_config(args, spec, rs, ndof, nvox, ws, safety):
    return {"workload": f"{args.config}: {spec.nx}x{spec.ny}x{spec.nz} voxels, {rs.c_rate}C charge, "
                        f"dt={rs.dt}s, plating on; one replica cell per GPU",
            "n_dof": ndof, "n_voxels": nvox,
            "l2": "flushed (256 MiB streamed read) before every timed step (value and e2e) and "
                  "every timed kernel launch",
            "parallelism": f"replicas x{ws}",
            "newton": ("Newton tol = max(1e-10, 1e-8 |F0|, cancellation floor) (BASELINE configs[2]); "
                       if args.config == "large" else
                       "Newton tol = max(1e-10, 1e-9 |F0|, cancellation floor) (reference defaults); ")
                      + (f"Krylov rtol 1e-10 on every Newton system" if safety == 0.0 else
                         f"Krylov rtol_k = max(1e-10, {safety} tol / |F_k|) (inexact Newton)"),
            "preconditioner": "multigrid values rebuilt at the first timed step (then every 32 "
                              "Newton solves and on dt changes)"}


def config0_line():
    """BASELINE configs[0] (tiny, 32x32x64, 10 steps at dt = 1 s) end to end through the
    public step API, beside the reference's own run of the same cell (fixture generation,
    tests/golden/make_golden_configs.py; measured in the build container, 1 core)."""
    import paper_1704_04139_b200 as P
    from paper_1704_04139_b200.microgen import generate_cell
    rs, spec = cell_for("tiny", 0)
    grid = generate_cell(spec)
    params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
    op = P.SystemOperator(P.build_dofmap(grid), params)
    mu = drive_mu(grid.labels, grid.voxel_size, rs.c_rate, params)
    cfg = P.SolverConfig(dt_init=min(0.05, rs.dt), dt_max=rs.dt)
    st = P.prepare_initial_state(op, params, mu, cfg)
    st, *_ = P.step(op, st, rs.dt, mu, cfg)       # warm
    t0 = time.perf_counter()
    for _ in range(rs.n_steps):
        st, *_ = P.step(op, st, rs.dt, mu, cfg)
    gpu = rs.n_steps / (time.perf_counter() - t0)
    out = {"workload": "tiny: 32x32x64, 1C, dt=1s, 10 steps (BASELINE configs[0])",
           "gpu_steps_per_s_step_api": gpu}
    fx = os.path.join(REPO, "tests", "golden", "config_tiny.npz")
    if os.path.exists(fx):
        with np.load(fx) as z:
            sec = float(z["ref_seconds"][1])
            n = int(z["n_steps"])
        out.update({"reference_steps_per_s": n / sec, "reference_cores": 1,
                    "reference_measured": "the reference package itself (SuperLU Newton) on the whole "
                                          "cell, unextrapolated, when its golden curves were generated "
                                          "(build container host, not this box)"})
    return out


def other_configs(args):
    """BASELINE configs[3] (batched study) and configs[4] (POD Gram + projection; ROM online
    stage) measured in the same run as the headline, with shortened step counts, so the
    driver's bench line carries them (each leg guarded: a failure is reported, not fatal)."""
    import copy
    out = {}
    legs = (("batched", run_batched, dict(steps=5, warmup=3)),
            ("pod", run_pod, dict(steps=3, warmup=1)),
            ("rom", run_rom, dict(steps=500, warmup=1)))
    for name, fn, over in legs:
        a = copy.copy(args)
        for k, v in over.items():
            setattr(a, k, v)
        a.config = name
        t0 = time.perf_counter()
        try:
            r = fn(a, 1, 0, int(os.environ.get("LOCAL_RANK", "0")))
            keep = ("metric", "value", "unit", "steps", "ms_per_step", "config", "roofline", "projection",
                    "krylov_iters_per_cell_step", "newton_iters_per_step", "parameter_batch",
                    "qoi_max_rel_dev_vs_fom_training_window", "offline", "max_rel_err_vs_cublas", "e2e")
            out[name] = {k: r[k] for k in keep if k in r}
        except Exception as e:  # noqa: BLE001
            out[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
        out[name]["wall_s"] = time.perf_counter() - t0
    return out


def run_ours(args, ws, rank, local):
    import torch
    import paper_1704_04139_b200 as P
    from paper_1704_04139_b200 import _dev, _native
    from paper_1704_04139_b200.microgen import generate_cell
    import ctypes

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rs, spec = cell_for(args.config, rank)
    grid = generate_cell(spec)
    params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
    dof = P.build_dofmap(grid)
    op = P.SystemOperator(dof, params)
    mu = drive_mu(grid.labels, grid.voxel_size, rs.c_rate, params)
    cfg = solver_config(P, args.config, rs, LINEAR_SAFETY)
    state = P.prepare_initial_state(op, params, mu, cfg)
    L = _native.lib()
    x0 = _dev.to_dev(state.x).clone()
    npl0 = _dev.to_dev(state.n_pl if state.n_pl.size else np.zeros(1)).clone()
    x, npl = x0.clone(), npl0.clone()
    c = cfg.to_c()
    st = _native.HcNewtonStats()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream or None

    def one_step(cc=c):
        _native.check(L.hc_step(op.native.handle, _dev.ptr(x), _dev.ptr(npl), 0.0, rs.dt, mu,
                                ctypes.byref(cc), ctypes.byref(st), sp))
        return st.n_iter, st.krylov_iters

    for _ in range(args.warmup):
        one_step()
    x_warm, npl_warm = x.clone(), npl.clone()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    newton, krylov = [], []
    n0 = ctypes.c_int64(0)
    _native.check(L.hc_launch_count(ctypes.byref(n0)))
    # the timed window pays at least one full multigrid rebuild (conservative for K < 32)
    _native.check(L.hc_precond_refresh(op.native.handle))
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for k in range(args.steps):
            _native.check(L.hc_flush_l2(L2_FLUSH_BYTES, sp))  # read-flush L2 between timed steps
            evs[k][0].record(stream)
            it, kr = one_step()
            evs[k][1].record(stream)
            newton.append(it)
            krylov.append(kr)
        torch.cuda.synchronize()
    n1 = ctypes.c_int64(0)
    _native.check(L.hc_launch_count(ctypes.byref(n1)))
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()

    # ---- e2e: the same K steps (from the same warm state) through the host-buffer entry
    # point: pinned H2D of the packed state + n_pl, step, D2H back, every step
    bi = (dof.n_total + max(dof.n_plated, 0)) * 8
    xh = torch.empty(dof.n_total, dtype=torch.float64).pin_memory()
    nh = torch.empty(max(dof.n_plated, 1), dtype=torch.float64).pin_memory()
    xh.copy_(x_warm.cpu())
    nh.copy_(npl_warm.cpu())
    stp = _native.HcNewtonStats()
    _native.check(L.hc_precond_refresh(op.native.handle))
    torch.cuda.synchronize()
    e2e_s = 0.0
    for _ in range(args.steps):
        _native.check(L.hc_flush_l2(L2_FLUSH_BYTES, sp))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _native.check(L.hc_step_host(op.native.handle, xh.data_ptr(), nh.data_ptr(), 0.0,
                                     rs.dt, mu, ctypes.byref(c), ctypes.byref(stp)))
        e2e_s += time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = ws * args.steps / e2e_s

    # ---- inexact Newton beside it (same warm state, same K): Krylov stops at
    # max(1e-10, 0.3 tol/|F_k|); whole-run curve parity against the exact path is tested
    inexact = None
    if rank == 0 and not args.no_inexact:
        ci = solver_config(P, args.config, rs, INEXACT_SAFETY).to_c()
        x.copy_(x_warm)
        npl.copy_(npl_warm)
        _native.check(L.hc_precond_refresh(op.native.handle))
        torch.cuda.synchronize()
        ms_i, kr_i = 0.0, 0
        for _ in range(args.steps):
            _native.check(L.hc_flush_l2(L2_FLUSH_BYTES, sp))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _, kr = one_step(ci)
            b.record(stream)
            b.synchronize()
            ms_i += a.elapsed_time(b)
            kr_i += kr
        inexact = {"linear_safety": INEXACT_SAFETY, "value": args.steps / (ms_i * 1e-3), "unit": "steps/s",
                   "krylov_iters_per_step": kr_i / args.steps,
                   "curve_parity": "tests/test_gpu_configs.py (whole run vs the exact-tolerance path "
                                   "and the reference fixtures, 1e-6)"}

    # ---- kernel timings: residual and J v at the trajectory's current state
    beta = rs.dt * op.face_area / params.constants.F
    kt = kernel_roofline(op, grid, params, x, npl, beta, rs.dt, args.config)
    ndof = dof.n_total
    nvox = int(op.native.info.n_vox)
    at_scale = None
    if rank == 0 and args.config != "large" and not args.no_at_scale:
        at_scale = roofline_at_scale()

    out = None
    if rank == 0:
        value = ws * args.steps / (total_ms * 1e-3)
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            vals, cores, sample = cpu_sample(args.config, rounds=1)
            cpu = {"value": vals[0], "unit": "steps/s", "cores": cores, "kind": "port",
                   "sample": sample}
        out = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded ball-union microstructure, BASELINE config shapes)",
            "config": workload_config(args, spec, rs, ndof, nvox, ws, LINEAR_SAFETY),
            "newton_iters_per_step": float(np.mean(newton)),
            "krylov_iters_per_step": float(np.mean(krylov)),
            # the full implicit step in DOF-updates/s (all ranks' cells)
            "dof_updates_per_s": value * ndof,
            "gdof_per_s": {"residual": ndof / (kt["res_ms"] * 1e-3) / 1e9,
                           "jvp": ndof / (kt["jv_ms"] * 1e-3) / 1e9},
            "kernel_ms": kt["kernel_ms"],
            "roofline": kt["roofline"],
            "roofline_at_scale": at_scale,
            "inexact_newton": inexact,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "steps/s", "h2d_bytes_per_step": bi,
                    "d2h_bytes_per_step": bi},
            "gpu_launches": int(n1.value - n0.value),
            "clocks": clk.summary(),
        }
        if not args.no_config0:
            out["config0"] = config0_line()
        if ws == 1 and not args.no_other_configs:
            out["other_configs"] = other_configs(args)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return out


def run_batched(args, ws, rank, local):
    """BASELINE config 3: 128 cells per GPU stepped concurrently (cell-steps/s)."""
    import torch
    import paper_1704_04139_b200 as P
    from paper_1704_04139_b200 import batch as B
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = args.cells
    cfg = P.SolverConfig(dt_init=1.0, dt_max=1.0, linear_safety=LINEAR_SAFETY)
    cells = B.make_batch(n, first_seed=100 + 1000 * rank, cfg=cfg)
    for _ in range(args.warmup):
        B.step_batch(cells, 1.0, cfg)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    iters = 0
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            st = B.step_batch(cells, 1.0, cfg)
            iters += sum(s.krylov_iters for s in st)
        torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([el], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        el = float(t.item())
        torch.distributed.destroy_process_group()
    if rank != 0:
        return None
    nd = sum(c.op.dof.n_total for c in cells)
    return {"metric": "batched parameter study: cell implicit steps/s", "value": ws * n * args.steps / el,
            "unit": "cell-steps/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cells 100+)",
            "config": {"workload": f"batched: {n} cells of 48x48x96 per GPU, per-cell C-rate / "
                       "kinetics / diffusivity / plating exchange drawn from the BASELINE ranges, dt=1s",
                       "n_dof_per_gpu": nd, "l2": "working set >> L2 (cells x ~100 MB)"},
            "krylov_iters_per_cell_step": iters / (n * args.steps), "clocks": clk.summary()}


def run_pod(args, ws, rank, local):
    """BASELINE config 4 offline stage: POD Gram S^T W S of 2.1M DOF x 400 snapshots and the
    rank-60 basis projection S (U / sigma), both on the FP64 tensor cores (DMMA)."""
    import torch
    from paper_1704_04139_b200 import _native, pod
    torch.cuda.set_device(local)
    n_dof, n_snap, rank_k = 2_100_000, 400, 60
    g = torch.Generator(device="cuda").manual_seed(7)
    # row-major (n_dof, n_snap): the snapshots of one DOF contiguous, as the ROM's snapshot
    # matrix is stored; the kernels read it in place
    S = torch.randn(n_dof, n_snap, device="cuda", dtype=torch.float64, generator=g)
    w = torch.rand(n_dof, device="cuda", dtype=torch.float64, generator=g) + 0.5
    U = torch.randn(n_snap, rank_k, device="cuda", dtype=torch.float64, generator=g)
    for _ in range(args.warmup):
        pod.pod_gram(S, w)
        pod.tc_matmul(S, U)
    torch.cuda.synchronize()

    def timed(fn):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        out = None
        for a, b in ev:
            _native.check(_native.lib().hc_flush_l2(L2_FLUSH_BYTES, torch.cuda.current_stream().cuda_stream))
            a.record()
            out = fn()
            b.record()
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev) / args.steps, out

    with ClockSampler(torch.cuda.current_device()) as clk:
        ms, G = timed(lambda: pod.pod_gram(S, w))
        ms_p, V = timed(lambda: pod.tc_matmul(S, U))
    peak = ctypes.c_double(0.0)
    _native.check(_native.lib().hc_dmma_peak(ctypes.byref(peak), None))
    # useful flops: the n (n + 1) / 2 distinct entries of the symmetric Gram, 2 flops per DOF
    flops = float(n_snap) * (n_snap + 1) * n_dof
    flops_p = 2.0 * n_dof * n_snap * rank_k
    ref = (S.t() * w) @ S
    err = float((G - ref).abs().max() / ref.abs().max())
    refp = S @ U
    err_p = float((V - refp).abs().max() / refp.abs().max())
    tf, tfp = flops / (ms * 1e-3) / 1e12, flops_p / (ms_p * 1e-3) / 1e12
    return {"metric": "POD snapshot Gram S^T W S (FP64 DMMA)", "value": tf * 1e3,
            "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic snapshots",
            "config": {"workload": f"pod: {n_dof} DOF x {n_snap} snapshots, rank {rank_k} projection",
                       "flops": "Gram: n_snap (n_snap + 1) n_dof (distinct entries of the symmetric "
                                "matrix, 2 flops each; the kernel computes upper-triangle tiles only)",
                       "l2": "flushed before every timed launch"},
            "roofline": {"bound": "tensor (FP64 DMMA)", "achieved": tf, "peak": peak.value,
                         "peak_kind": "measured (hc_dmma_peak: register-only DMMA probe)", "unit": "TFLOP/s",
                         "frac": tf / peak.value if peak.value else None, "traffic": None},
            "projection": {"what": "S (U / sigma): 2.1M x 400 times 400 x 60 (hc_dgemm)", "ms": ms_p,
                           "tflops": tfp, "frac_of_dmma_peak": tfp / peak.value if peak.value else None,
                           "max_rel_err_vs_cublas": err_p},
            "max_rel_err_vs_cublas": err, "clocks": clk.summary()}


def run_rom(args, ws, rank, local):
    """BASELINE config 4 end to end on the medium cell: full-order snapshots, POD (DMMA
    Gram) per field, EI (DEIM) rows of the nonlinear sub-operators, projection, then the
    reduced Newton solve for 500 steps in one kernel launch (timed, CUDA events)."""
    import torch
    import paper_1704_04139_b200 as P
    from paper_1704_04139_b200 import mor
    from paper_1704_04139_b200.microgen import generate_cell
    from paper_1704_04139_b200.qoi import qoi_vectors
    torch.cuda.set_device(local)
    rs, spec = cell_for("medium", rank)
    grid = generate_cell(spec)
    params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
    op = P.SystemOperator(P.build_dofmap(grid), params)
    mu = drive_mu(grid.labels, grid.voxel_size, rs.c_rate, params)
    dt = rs.dt
    cfg = P.SolverConfig(dt_init=min(0.05, dt), dt_max=dt, linear_safety=LINEAR_SAFETY)
    st = P.prepare_initial_state(op, params, mu, cfg)
    tt = {}
    t0 = time.perf_counter()
    snaps = mor.collect_snapshots(op, st.x, st.n_pl, mu, dt, args.rom_snapshots,
                                  P.SolverConfig(dt_init=dt, dt_max=dt, linear_safety=0.0))
    torch.cuda.synchronize()
    tt["snapshots_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rom = mor.build_rom(op, snaps, args.rom_rank, args.rom_rank, args.rom_ei)
    torch.cuda.synchronize()
    tt["offline_build_s"] = time.perf_counter() - t0
    xt0 = rom.project(st.x)
    n_steps = args.rom_steps
    for _ in range(max(1, args.warmup)):
        mor.solve_rom(op, rom, xt0, st.n_pl, mu, dt, 2)
    n0 = ctypes.c_int64(0)
    from paper_1704_04139_b200 import _native
    _native.check(_native.lib().hc_launch_count(ctypes.byref(n0)))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        a.record()
        tr = mor.solve_rom(op, rom, xt0, st.n_pl, mu, dt, n_steps)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    n1 = ctypes.c_int64(0)
    _native.check(_native.lib().hc_launch_count(ctypes.byref(n1)))
    # e2e: host reduced state in, QoI curves out, through the public API
    # the MOR use case: many applied currents at once, one thread-block cluster each
    n_par = args.rom_batch
    mus = mu * np.linspace(0.5, 1.0, n_par)
    mor.solve_rom_batch(op, rom, xt0, st.n_pl, mus[:2], dt, 2)
    torch.cuda.synchronize()
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record()
    mor.solve_rom_batch(op, rom, xt0, st.n_pl, mus, dt, n_steps)
    b2.record()
    torch.cuda.synchronize()
    batch_ms = a2.elapsed_time(b2)
    xh = xt0.cpu().numpy()
    t0 = time.perf_counter()
    tr2 = mor.solve_rom(op, rom, xh, st.n_pl, mu, dt, n_steps)
    v_host = np.asarray(tr2.voltage)
    e2e_s = time.perf_counter() - t0
    v_cp, v_ac = qoi_vectors(op.dof)
    X = snaps.X.cpu().numpy()
    nt = min(n_steps, X.shape[1] - 1)
    fom_v = v_cp @ X[:, 1:nt + 1]
    dev_v = float(np.max(np.abs(tr.voltage[:nt] - fom_v)) / np.max(np.abs(fom_v)))
    return {"metric": "reduced implicit time steps/s (ROM online stage, config 4)",
            "value": n_steps / (ms * 1e-3), "unit": "steps/s", "n_gpus": 1, "steps": n_steps,
            "warmup": args.warmup, "ms_per_step": ms / n_steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (medium cell, seeded ball-union microstructure)",
            "config": {"workload": f"rom: medium cell {spec.nx}x{spec.ny}x{spec.nz}, {args.rom_snapshots} "
                                   f"full-order snapshots, POD rank {rom.k_c}+{rom.k_p}, {rom.m} EI rows, "
                                   f"{n_steps} reduced steps at dt={dt}s", "n_dof": op.dof.n_total,
                       "stencil_dofs": rom.dims["n_s"], "active_faces": rom.dims["n_f"]},
            "newton_iters_per_step": float(np.mean(tr.newton_iters)),
            "offline": tt,
            "qoi_max_rel_dev_vs_fom_training_window": dev_v,
            "parameter_batch": {"n_params": n_par, "mu_range": [float(mus.min()), float(mus.max())],
                                "reduced_steps_per_s": n_par * n_steps / (batch_ms * 1e-3),
                                "ms": batch_ms},
            "e2e": {"value": n_steps / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": 8 * rom.k / n_steps,
                    "d2h_bytes_per_step": 16.0},
            "gpu_launches": int(n1.value - n0.value),
            "roofline": {"bound": "latency (one thread-block cluster; k=%d dense LU per step)" % rom.k, "achieved": None,
                         "peak": None, "unit": None, "frac": None, "traffic": None},
            "clocks": clk.summary()}


def run_reference(args, ws, rank):
    if rank != 0:
        return None
    from paper_1704_04139_b200.configs import CONFIGS
    vals, cores, sample = cpu_sample(args.config, rounds=args.steps, warmup=args.warmup)
    total_s = sum(1.0 / v for v in vals)
    value = len(vals) / total_s
    from paper_1704_04139_b200.microgen import generate_cell
    rs, spec = cell_for(args.config, 0)
    lab = generate_cell(spec).labels
    nvox = int(lab.size)
    # DOF count of the same cell (dofmap.py:71-101): c on graphite + electrolyte voxels, phi
    # on every voxel but the grounded counter-collector layer
    n_dof = int(np.count_nonzero(np.isin(lab, (0, 1)))) + nvox - int(np.count_nonzero(lab[-1] == 5))
    # the same config object as the GPU arm: the workload is the same cell; how the CPU
    # number was obtained (column samples, extrapolated) is in cpu_baseline.sample
    cfg = workload_config(args, spec, rs, n_dof, nvox, ws, LINEAR_SAFETY)
    return {"metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded ball-union microstructure, BASELINE config shapes)",
            "config": cfg, "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="large")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-at-scale", action="store_true", help="skip the large-grid kernel roofline")
    ap.add_argument("--no-inexact", action="store_true", help="skip the inexact-Newton figure")
    ap.add_argument("--no-config0", action="store_true", help="skip the tiny-config line")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the batched / POD / ROM legs appended to the headline line")
    ap.add_argument("--cells", type=int, default=128)
    ap.add_argument("--rom-snapshots", type=int, default=400)
    ap.add_argument("--rom-rank", type=int, default=60)
    ap.add_argument("--rom-ei", type=int, default=300)
    ap.add_argument("--rom-steps", type=int, default=500)
    ap.add_argument("--rom-batch", type=int, default=64)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    ws, rank, local = dist_env()
    if args.impl == "reference":
        out = run_reference(args, ws, rank)
    elif args.config == "batched":
        out = run_batched(args, ws, rank, local)
    elif args.config == "pod":
        out = run_pod(args, ws, rank, local)
    elif args.config == "rom":
        out = run_rom(args, ws, rank, local)
    else:
        out = run_ours(args, ws, rank, local)
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
