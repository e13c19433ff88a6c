"""Whole-run golden curves of the BASELINE configurations, produced by the REFERENCE.

    python tests/golden/make_golden_configs.py [tiny] [batch0 batch1 batch2]

Build container only (needs /root/reference/pkg/src); the GPU box reads the
committed ``.npz`` files.  Each case runs the reference's own public API
(``prepare_initial_state`` + ``step`` of fvm/timestepping.py:64-114, QoIs of
fvm/qoi.py:37-44) with SuperLU Newton (fvm/newton.py:75-77) on a cell built by
this package's seeded generator (``generate_cell``; the labels are stored and a
CPU test checks the generator still reproduces them bit for bit):

* ``tiny``   — BASELINE configs[0]: 32x32x64, 1C charge, dt = 1 s, 10 steps,
  plating exchange current 1e-3 A/m^2;
* ``batchK`` — BASELINE configs[3]: cell K (seed 100 + K) of the 48x48x96 batched
  parameter study with its sampled per-cell parameters (batch.sample_parameters),
  dt = 1 s, 2 steps.

Stored per case: labels, the run settings, per-step voltage / mean solid
concentration / plated inventory / Newton iterations, and at two trajectory
states (after the first and the last step) the state, the operator value
``apply(x, n_pl, mu, beta)`` and ``(J + diag(1/dt on c rows)) v`` for a seeded v.
"""

from __future__ import annotations

import dataclasses
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def _setup_paths():
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, REPO)


def case_settings(name: str):
    """(CellSpec, reference MaterialParams kwargs, mu recipe, dt, n_steps) of a case."""
    from paper_1704_04139_b200 import batch as B
    from paper_1704_04139_b200.configs import CONFIGS
    if name == "tiny":
        rs = CONFIGS["tiny"]
        kw = dict(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
        return rs.cell, kw, rs.c_rate, rs.dt, rs.n_steps
    k = int(name[len("batch"):])
    pr = B.sample_parameters(k + 1)[k]
    spec = dataclasses.replace(B.BATCH_SPEC, seed=100 + k)
    kw = dict(soc_init=0.1, i00_grel_scale=pr["i00_grel_scale"], d_el_scale=pr["d_el_scale"],
              i00_plel=pr["plating_exchange"] / np.sqrt(1000.0))
    return spec, kw, pr["c_rate"], 1.0, 2


def run_case(name: str):
    _setup_paths()
    from halfcell.echem import MaterialParams as RefParams
    from halfcell.fvm import (SolverConfig, SystemOperator, build_dofmap, prepare_initial_state,
                              qoi_cell_voltage, qoi_mean_solid_conc, step)
    from halfcell.microgen import PhaseGrid
    from paper_1704_04139_b200.microgen import generate_cell

    spec, kw, c_rate, dt, n_steps = case_settings(name)
    kw = dict(kw)
    base = RefParams()
    gs = kw.pop("i00_grel_scale", 1.0)
    ds = kw.pop("d_el_scale", 1.0)
    params = RefParams(i00_grel=base.i00_grel * gs, d_el=base.d_el * ds, **kw)
    g = generate_cell(spec)
    labels = g.labels
    grid = PhaseGrid(labels, g.voxel_size)
    dof = build_dofmap(grid)
    op = SystemOperator(dof, params)
    h = g.voxel_size * 1e-6
    vol = float(np.count_nonzero(labels == 1)) * h ** 3
    mu = -c_rate * params.c_gr_max * params.constants.F * vol / 3600.0 / (spec.nx * spec.ny * h * h)
    cfg = SolverConfig(dt_init=min(0.05, dt), dt_max=dt)
    t0 = time.perf_counter()
    state = prepare_initial_state(op, params, mu, cfg)
    t_init = time.perf_counter() - t0
    beta = cfg.strip_beta(op, dt)
    rng = np.random.default_rng(23)
    v = rng.standard_normal(dof.n_total)
    mass = np.zeros(dof.n_total)
    mass[: dof.n_c] = 1.0 / dt
    V, C, N, IT, DT = ([qoi_cell_voltage(state, dof)], [qoi_mean_solid_conc(state, dof)],
                       [float(state.n_pl.sum())], [], [])
    out = dict(labels=labels, voxel_size=g.voxel_size, mu=mu, dt=dt, beta=beta, n_steps=n_steps,
               c_rate=c_rate, soc_init=params.soc_init, i00_grel=params.i00_grel,
               d_el=params.d_el, i00_plel=params.i00_plel, v=v,
               spec=np.array(repr(spec)), x0=state.x, npl0=state.n_pl)
    t0 = time.perf_counter()
    for k in range(1, n_steps + 1):
        state, dt_used, _, info = step(op, state, dt, mu, cfg)
        V.append(qoi_cell_voltage(state, dof))
        C.append(qoi_mean_solid_conc(state, dof))
        N.append(float(state.n_pl.sum()))
        IT.append(info.n_iter)
        DT.append(dt_used)
        if k in (1, n_steps):
            tag = "first" if k == 1 else "last"
            J = op.jacobian(state.x, state.n_pl, mu, beta=beta)
            out[f"x_{tag}"] = state.x
            out[f"npl_{tag}"] = state.n_pl
            out[f"apply_{tag}"] = op.apply(state.x, state.n_pl, mu, beta=beta)
            out[f"jv_{tag}"] = J @ v + mass * v
        print(f"{name}: step {k} dt={dt_used} newton={info.n_iter} V={V[-1]:.12f} "
              f"({time.perf_counter() - t0:.0f} s)", flush=True)
    out.update(voltage=np.array(V), mean_c=np.array(C), npl_sum=np.array(N),
               newton_iters=np.array(IT), dts=np.array(DT),
               ref_seconds=np.array([t_init, time.perf_counter() - t0]))
    path = os.path.join(HERE, f"config_{name}.npz")
    np.savez_compressed(path, **out)
    print(name, labels.shape, dof.describe(), "->", os.path.getsize(path), "bytes", flush=True)
    return name


def main():
    names = sys.argv[1:] or ["tiny", "batch0", "batch1", "batch2"]
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    with mp.get_context("spawn").Pool(len(names)) as pool:
        for n in pool.imap_unordered(run_case, names):
            print("done", n, flush=True)


if __name__ == "__main__":
    main()
