"""GPU: time-step control semantics of the reference (timestepping.py:64-176):
retry with a halved step on Newton failure, SimulationError at dt_min, schedule
knots hit exactly, run_transient trajectory bookkeeping."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _small():
    import paper_1704_04139_b200 as P
    g = np.load("tests/golden/refgen_10x10x20.npz")
    params = P.MaterialParams()
    grid = P.PhaseGrid(g["labels"], float(g["voxel_size"]))
    op = P.SystemOperator(P.build_dofmap(grid), params)
    return P, grid, params, op


def test_retry_halves_the_step_when_newton_fails():
    P, grid, params, op = _small()
    cfg_ok = P.SolverConfig()
    st = P.prepare_initial_state(op, params, -20.0, cfg_ok)
    # a one-iteration Newton budget fails at dt = 2 s but a smaller step converges
    cfg = P.SolverConfig(newton_max_iter=1, dt_init=0.05, dt_min=1e-6, dt_max=2.5)
    new, dt_used, dt_next, info = P.step(op, st, 2.0, -20.0, cfg)
    assert info.retries >= 1
    assert dt_used == pytest.approx(2.0 * 0.5 ** info.retries)
    assert new.t == pytest.approx(st.t + dt_used)
    assert np.all(new.n_pl >= 0.0)


def test_time_step_underflow_raises_simulation_error():
    P, grid, params, op = _small()
    st = P.prepare_initial_state(op, params, -20.0, P.SolverConfig())
    cfg = P.SolverConfig(newton_max_iter=0, dt_init=0.5, dt_min=0.25, dt_max=2.5)
    with pytest.raises(P.SimulationError, match="time step underflow"):
        P.step(op, st, 1.0, -20.0, cfg)


def test_run_transient_schedule_and_adaptive():
    P, grid, params, op = _small()
    drive = P.BoundaryDrive(-20.0)
    cfg = P.SolverConfig(dt_init=0.1, dt_max=1.0)
    traj = P.run_transient(grid, params, drive, cfg, 2.0, schedule=np.array([0.5, 1.0, 2.0]), op=op)
    assert np.allclose(traj.times, [0.0, 0.5, 1.0, 2.0])
    traj2 = P.run_transient(grid, params, drive, cfg, 1.0, op=op)
    assert traj2.times[-1] == pytest.approx(1.0)
    assert all(np.diff(traj2.times) > 0)
    # the adaptive step grows by grow_factor while Newton is easy, capped at dt_max
    assert max(traj2.dts) <= cfg.dt_max + 1e-12
