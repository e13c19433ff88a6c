"""Damped Newton for the implicit-Euler systems, on the GPU.

Mirrors ``halfcell.fvm.newton`` (reference ``src/halfcell/fvm/newton.py``):
``SolverConfig`` with the same fields and validation, ``newton_solve`` and
``solve_initial_potential`` with the same signatures, tolerance rule
``max(atol, rtol |F(x0)|, cancellation floor)``, positivity guard and
residual-halving line search.  The linear systems are solved on the device by
BiCGStab preconditioned with the field-split aggregation multigrid
(``csrc/hc_amg.cu``); ``linear_solver`` is accepted for compatibility and
both values select that device solver.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _native
from .errors import ConfigError


@dataclass
class SolverConfig:
    newton_rtol: float = 1e-9
    newton_atol: float = 1e-10
    newton_max_iter: int = 20
    linear_solver: str = "direct"
    linear_rtol: float = 1e-10
    dt_init: float = 0.05
    dt_min: float = 1e-6
    dt_max: float = 2.5
    grow_factor: float = 1.2
    shrink_factor: float = 0.5
    easy_iter_threshold: int = 5
    implicit_plated: bool = True
    krylov_max_iter: int = 1000
    # Krylov tolerance per Newton iteration: max(linear_rtol, linear_safety * tol / |F_k|)
    # (the linear solve never goes beyond what the Newton tolerance can use); 0 disables
    linear_safety: float = 0.0

    def __post_init__(self):
        if not 0.0 < self.shrink_factor < 1.0 < self.grow_factor:
            raise ConfigError("need 0 < shrink_factor < 1 < grow_factor")
        if not self.dt_min <= self.dt_init <= self.dt_max:
            raise ConfigError("need dt_min <= dt_init <= dt_max")
        if self.linear_solver not in ("direct", "krylov"):
            raise ConfigError("linear_solver must be 'direct' or 'krylov'")

    def strip_beta(self, op, dt: float) -> float:
        if not self.implicit_plated:
            return 0.0
        return dt * op.face_area / op.p.constants.F

    def to_c(self) -> _native.HcSolverConfig:
        c = _native.HcSolverConfig()
        c.newton_rtol = self.newton_rtol
        c.newton_atol = self.newton_atol
        c.newton_max_iter = self.newton_max_iter
        c.krylov_max_iter = self.krylov_max_iter
        c.linear_rtol = self.linear_rtol
        c.dt_init, c.dt_min, c.dt_max = self.dt_init, self.dt_min, self.dt_max
        c.grow_factor, c.shrink_factor = self.grow_factor, self.shrink_factor
        c.easy_iter_threshold = self.easy_iter_threshold
        c.implicit_plated = 1 if self.implicit_plated else 0
        c.linear_safety = self.linear_safety
        return c


@dataclass
class NewtonResult:
    x: np.ndarray
    iterates: list = field(default_factory=list)
    n_iter: int = 0
    residual_norms: list = field(default_factory=list)
    krylov_iters: int = 0


def newton_solve(op, x_guess, dt: float, x_prev, n_pl, mu: float, cfg: SolverConfig,
                 source=None) -> NewtonResult:
    """Solve ``m (x - x_prev)/dt + A(x; mu) + source = 0`` (reference ``newton.py:86-168``).

    Returns every accepted iterate (``NewtonResult.iterates``, the snapshot source of the
    reduction stage) and every residual norm, like the reference.  Inputs may be numpy
    arrays or CUDA tensors; outputs follow ``x_guess``.
    """
    if dt <= 0:
        raise ValueError("dt must be positive")
    n = op.dof.n_total
    xg, xp = _dev.to_dev(x_guess), _dev.to_dev(x_prev)
    nd = _dev.to_dev(n_pl) if _dev.numel(n_pl) else _dev.to_dev(np.zeros(1))
    src = _dev.to_dev(source) if source is not None else None
    out = _dev.empty(n)
    m = int(cfg.newton_max_iter)
    its = _dev.torch().empty((max(m, 1), n), dtype=_dev.torch().float64, device="cuda")
    norms = (ctypes.c_double * (m + 1))()
    st = _native.HcNewtonStats()
    c = cfg.to_c()
    _native.check(_native.lib().hc_newton_solve_ex(
        op.native.handle, _dev.ptr(xg), float(dt), _dev.ptr(xp), _dev.ptr(nd), float(mu), ctypes.byref(c),
        _dev.ptr(src) if src is not None else None, _dev.ptr(its), m, norms, m + 1, _dev.ptr(out),
        ctypes.byref(st), _dev.stream()))
    k = int(st.n_iter)
    x = _dev.like_input(out, x_guess)
    iterates = [_dev.like_input(its[i], x_guess) for i in range(k)]
    return NewtonResult(x, iterates, k, [float(norms[i]) for i in range(k + 1)], int(st.krylov_iters))


def solve_initial_potential(op, x0, n_pl, mu: float, cfg: SolverConfig):
    """Stationary potential solve at frozen c (reference ``newton.py:171-206``)."""
    xd = _dev.to_dev(x0)
    nd = _dev.to_dev(n_pl) if _dev.numel(n_pl) else _dev.to_dev(np.zeros(1))
    out = _dev.empty(op.dof.n_total)
    st = _native.HcNewtonStats()
    c = cfg.to_c()
    _native.check(_native.lib().hc_solve_initial_potential(op.native.handle, _dev.ptr(xd),
                                                           _dev.ptr(nd), float(mu),
                                                           ctypes.byref(c), _dev.ptr(out),
                                                           ctypes.byref(st), _dev.stream()))
    return _dev.like_input(out, x0)
