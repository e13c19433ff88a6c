"""Batched parameter study (BASELINE config 3): many independent cells resident on
one GPU, stepped concurrently through ``hc_step_batch`` (one private CUDA stream
per cell, host threads drive the per-cell Newton control).

This is the model-order-reduction use case of arXiv 1704.04139 (repeated
full-order solves over a parameter domain); the per-cell physics and step
semantics are exactly those of ``timestepping.step`` (reference
``fvm/timestepping.py:64-106``).
"""

from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass

import numpy as np

from . import _dev, _native
from .dofmap import build_dofmap
from .microgen import CellSpec, generate_cell
from .newton import SolverConfig
from .params import MaterialParams
from .system_operator import SystemOperator
from .timestepping import prepare_initial_state

BATCH_SPEC = CellSpec(48, 48, 96, 42, 12, seed=100, radius_mean=6.0, porosity=0.35)


@dataclass
class BatchCell:
    op: SystemOperator
    params: MaterialParams
    c_rate: float
    mu: float
    x: object          # CUDA fp64 tensor, packed state
    n_pl: object       # CUDA fp64 tensor
    t: float = 0.0


def sample_parameters(n: int, seed: int = 2017):
    """Per-cell study parameters, uniform over the BASELINE config-3 ranges."""
    rng = np.random.default_rng(seed)
    return [dict(c_rate=float(rng.uniform(0.5, 4.0)),
                 i00_grel_scale=float(rng.uniform(0.5, 2.0)),
                 d_el_scale=float(rng.uniform(0.5, 2.0)),
                 plating_exchange=float(rng.uniform(1e-4, 1e-2))) for _ in range(n)]


def charge_current(labels, voxel_um, c_rate, p: MaterialParams) -> float:
    h = voxel_um * 1e-6
    vol = float(np.count_nonzero(labels == 1)) * h ** 3
    area = labels.shape[1] * labels.shape[2] * h * h
    return -c_rate * p.c_gr_max * p.constants.F * vol / 3600.0 / area


def make_batch(n_cells: int = 128, first_seed: int = 100, spec: CellSpec = BATCH_SPEC,
               cfg: SolverConfig | None = None, soc_init: float = 0.1) -> list[BatchCell]:
    cfg = cfg or SolverConfig()
    cells = []
    for k, pr in enumerate(sample_parameters(n_cells)):
        grid = generate_cell(dataclasses.replace(spec, seed=first_seed + k))
        base = MaterialParams()
        p = MaterialParams(soc_init=soc_init, i00_grel=base.i00_grel * pr["i00_grel_scale"],
                           d_el=base.d_el * pr["d_el_scale"],
                           i00_plel=pr["plating_exchange"] / np.sqrt(base.c_el_init))
        op = SystemOperator(build_dofmap(grid), p)
        mu = charge_current(grid.labels, grid.voxel_size, pr["c_rate"], p)
        st = prepare_initial_state(op, p, mu, cfg)
        cells.append(BatchCell(op, p, pr["c_rate"], mu, _dev.to_dev(st.x).clone(),
                               _dev.to_dev(st.n_pl if st.n_pl.size else np.zeros(1)).clone()))
    return cells


def step_batch(cells: list[BatchCell], dt: float, cfg: SolverConfig, n_threads: int | None = None):
    """One accepted implicit step for every cell (concurrently on the device)."""
    import os
    n = len(cells)
    if n_threads is None:
        n_threads = int(os.environ.get("HC_BATCH_THREADS", "16"))
    ops = (ctypes.c_void_p * n)(*[c.op.native.handle.value for c in cells])
    xs = (ctypes.c_void_p * n)(*[c.x.data_ptr() for c in cells])
    ns = (ctypes.c_void_p * n)(*[c.n_pl.data_ptr() for c in cells])
    dts = (ctypes.c_double * n)(*([float(dt)] * n))
    mus = (ctypes.c_double * n)(*[c.mu for c in cells])
    stats = (_native.HcNewtonStats * n)()
    cc = cfg.to_c()
    _dev.torch().cuda.synchronize()
    code = _native.lib().hc_step_batch(ops, n, xs, ns, dts, mus, ctypes.byref(cc), stats, int(n_threads))
    # cells that stepped advance their clock even when another cell failed (a failed cell
    # keeps its input state; stats[i].status carries its error code)
    for c, s in zip(cells, stats):
        if s.status == 0:
            c.t += s.dt_used
    _native.check(code)
    return list(stats)
