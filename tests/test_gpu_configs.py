"""Parity on the BASELINE configurations (whole runs), through the C ABI.

* configs[0] (tiny, 32x32x64, 1C, dt = 1 s, 10 steps) and three cells of configs[3]
  (batched study, 48x48x96, their sampled per-cell parameters, 2 steps): voltage,
  mean solid concentration and plated inventory over the WHOLE run against the
  reference's own run (fixtures from tests/golden/make_golden_configs.py), with the
  exact (Krylov 1e-10) and the inexact-Newton (0.3) linear tolerance; residual and
  J v at two trajectory states of the reference run; the batch through ``hc_step_batch``.
* configs[1] / configs[2] (medium, large): residual and J v against the CPU oracle at
  real trajectory states; the inexact-Newton curves against the exact-tolerance path
  over the whole run (large: all 200 steps at Newton 1e-8 / Krylov 1e-10).

Bars (BASELINE north_star): residual and J v within 1e-10 relative per row (relative to
the sum of |contributions| of the row); curves within 1e-6 relative.
"""

import dataclasses

import numpy as np
import pytest

from conftest import config_cases, load_golden, scaled_err
from oracle import fvm_oracle as O

pytestmark = pytest.mark.gpu

TOL_RES = 1e-10
TOL_CURVE = 1e-6


def _P():
    import paper_1704_04139_b200 as P
    return P


def _params(g):
    P = _P()
    return P.MaterialParams(soc_init=float(g["soc_init"]), i00_grel=float(g["i00_grel"]),
                            d_el=float(g["d_el"]), i00_plel=float(g["i00_plel"]))


def _oracle(g):
    p = O.Params(soc_init=float(g["soc_init"]), i00_grel=float(g["i00_grel"]), d_el=float(g["d_el"]),
                 i00_plel=float(g["i00_plel"]))
    return O.OracleOperator(g["labels"], float(g["voxel_size"]), p)


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


@pytest.fixture(scope="module", params=config_cases())
def cfgcase(request):
    P = _P()
    g = load_golden(f"config_{request.param}")
    params = _params(g)
    dof = P.build_dofmap(P.PhaseGrid(g["labels"], float(g["voxel_size"])))
    return request.param, g, P.SystemOperator(dof, params), dof, params


@pytest.mark.parametrize("which", ["first", "last"])
def test_residual_and_jv_at_reference_trajectory_states(cfgcase, which):
    """apply(x, n_pl, mu, beta) and (J + diag(1/dt on c)) v at the reference's own states
    after the first and the last step of its run."""
    name, g, op, dof, _ = cfgcase
    orc = _oracle(g)
    x, npl = g[f"x_{which}"], g[f"npl_{which}"]
    mu, beta, dt, v = float(g["mu"]), float(g["beta"]), float(g["dt"]), g["v"]
    r = op.apply(x, npl, mu, beta=beta)
    assert scaled_err(r, g[f"apply_{which}"], orc.row_scale(x, npl, mu, beta)) < TOL_RES
    J = orc.jacobian(x, npl, beta)
    mass = np.zeros(dof.n_total)
    mass[: dof.n_c] = 1.0 / dt
    jv = op.jvp(x, npl, v, beta=beta, inv_dt=1.0 / dt)
    assert scaled_err(jv, g[f"jv_{which}"], abs(J) @ np.abs(v) + mass * np.abs(v)) < TOL_RES


def _curves_step_api(op, dof, params, g, safety):
    P = _P()
    mu, dt, n = float(g["mu"]), float(g["dt"]), int(g["n_steps"])
    cfg = P.SolverConfig(dt_init=min(0.05, dt), dt_max=dt, linear_safety=safety)
    st = P.prepare_initial_state(op, params, mu, cfg)
    V, C, N = [P.qoi_cell_voltage(st, dof)], [P.qoi_mean_solid_conc(st, dof)], [float(st.n_pl.sum())]
    for _ in range(n):
        st, dt_used, _, info = P.step(op, st, dt, mu, cfg)
        assert dt_used == pytest.approx(dt) and info.retries == 0
        V.append(P.qoi_cell_voltage(st, dof))
        C.append(P.qoi_mean_solid_conc(st, dof))
        N.append(float(st.n_pl.sum()))
    return np.array(V), np.array(C), np.array(N)


@pytest.mark.parametrize("safety", [0.0, 0.3])
def test_whole_run_curves_vs_reference(cfgcase, safety):
    """Every step of the config's run: cell voltage, mean solid concentration and plated
    inventory within 1e-6 of the reference's run (fvm/timestepping.py:64-106, qoi.py:37-44)."""
    name, g, op, dof, params = cfgcase
    V, C, N = _curves_step_api(op, dof, params, g, safety)
    assert V.size == g["voltage"].size
    assert _rel(V, g["voltage"]) < TOL_CURVE
    assert _rel(C, g["mean_c"]) < TOL_CURVE
    assert np.allclose(N, g["npl_sum"], rtol=TOL_CURVE, atol=1e-6 * float(np.max(g["npl_sum"])))


def test_batched_cells_vs_reference():
    """configs[3]: the reference-pinned cells stepped TOGETHER through hc_step_batch (the
    batched path, device-resident Newton), each against its own reference run."""
    P = _P()
    from paper_1704_04139_b200 import _dev
    from paper_1704_04139_b200 import batch as B
    names = [n for n in config_cases() if n.startswith("batch")]
    if not names:
        pytest.skip("no batch fixtures")
    cells, gs = [], []
    cfg = P.SolverConfig(dt_init=1.0, dt_max=1.0)
    for n in names:
        g = load_golden(f"config_{n}")
        params = _params(g)
        op = P.SystemOperator(P.build_dofmap(P.PhaseGrid(g["labels"], float(g["voxel_size"]))), params)
        st = P.prepare_initial_state(op, params, float(g["mu"]), cfg)
        assert _rel(P.qoi_cell_voltage(st, op.dof), g["voltage"][0]) < TOL_CURVE
        cells.append(B.BatchCell(op, params, float(g["c_rate"]), float(g["mu"]), _dev.to_dev(st.x).clone(),
                                 _dev.to_dev(st.n_pl if st.n_pl.size else np.zeros(1)).clone()))
        gs.append(g)
    for k in range(1, int(gs[0]["n_steps"]) + 1):
        stats = B.step_batch(cells, 1.0, cfg)
        for c, g, s in zip(cells, gs, stats):
            assert s.status == 0 and s.dt_used == 1.0
            v_cp, v_ac = P.qoi_vectors(c.op.dof)
            x = c.x.cpu().numpy()
            assert _rel(v_cp @ x, g["voltage"][k]) < TOL_CURVE
            assert _rel(v_ac @ x, g["mean_c"][k]) < TOL_CURVE
            npl = float(c.n_pl.sum()) if c.op.dof.n_plated else 0.0
            assert npl == pytest.approx(float(g["npl_sum"][k]), rel=TOL_CURVE, abs=1e-30)
    for c in cells:
        assert c.t == pytest.approx(int(gs[0]["n_steps"]))


# ------------------------------------------------------------------ medium / large
def _config_run(name, n_steps, safety, keep=()):
    """Fixed-dt run of a BASELINE config on the device; returns QoI curves and the states
    after the steps listed in ``keep``."""
    P = _P()
    from paper_1704_04139_b200.configs import CONFIGS
    from paper_1704_04139_b200.microgen import generate_cell
    rs = CONFIGS[name]
    grid = generate_cell(rs.cell)
    params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
    op = P.SystemOperator(P.build_dofmap(grid), params)
    h = grid.voxel_size * 1e-6
    mu = -rs.c_rate * params.c_gr_max * params.constants.F * np.count_nonzero(grid.labels == 1) * h ** 3 \
        / 3600.0 / (grid.labels.shape[1] * grid.labels.shape[2] * h * h)
    kw = dict(newton_rtol=1e-8, linear_rtol=1e-10) if name == "large" else {}
    cfg = P.SolverConfig(dt_init=min(0.05, rs.dt), dt_max=rs.dt, linear_safety=safety, **kw)
    st = P.prepare_initial_state(op, params, mu, cfg).to_device()
    dof = op.dof
    V, C, N, kept = [], [], [], {}
    for k in range(1, n_steps + 1):
        st, dt_used, _, info = P.step(op, st, rs.dt, mu, cfg)
        assert dt_used == pytest.approx(rs.dt) and info.retries == 0
        V.append(P.qoi_cell_voltage(st, dof))
        C.append(P.qoi_mean_solid_conc(st, dof))
        N.append(float(st.n_pl.sum()) if dof.n_plated else 0.0)
        if k in keep:
            kept[k] = st.to_host()
    return dict(op=op, grid=grid, params=params, mu=mu, dt=rs.dt, V=np.array(V), C=np.array(C),
                N=np.array(N), kept=kept)


@pytest.mark.parametrize("name,k", [("medium", 6), ("large", 3)])
def test_residual_and_jv_vs_oracle_at_trajectory_state(name, k):
    run = _config_run(name, k, 0.3, keep=(k,))
    op, grid, st = run["op"], run["grid"], run["kept"][k]
    P = run["params"]
    orc = O.OracleOperator(grid.labels, grid.voxel_size, O.Params(P))
    x, npl, mu, dt = st.x, st.n_pl, run["mu"], run["dt"]
    beta = dt * orc.face_area / orc.p.F
    r = op.apply(x, npl, mu, beta=beta)
    assert scaled_err(r, orc.apply(x, npl, mu, beta), orc.row_scale(x, npl, mu, beta)) < TOL_RES
    v = np.random.default_rng(3).standard_normal(x.size)
    J = orc.jacobian(x, npl, beta)
    assert scaled_err(op.jvp(x, npl, v, beta=beta), J @ v, abs(J) @ np.abs(v)) < TOL_RES


@pytest.mark.parametrize("name,n", [("medium", 20), ("large", 200)])
def test_inexact_newton_whole_run_matches_exact(name, n):
    """The inexact-Newton linear tolerance (Krylov stops at max(1e-10, 0.3 tol/|F_k|)) keeps
    the whole run's curves within 1e-6 of the exact-tolerance path (Krylov 1e-10 on every
    Newton system; large: BASELINE's Newton 1e-8 / Krylov 1e-10, all 200 steps)."""
    a = _config_run(name, n, 0.0)
    b = _config_run(name, n, 0.3)
    assert _rel(b["V"], a["V"]) < TOL_CURVE
    assert _rel(b["C"], a["C"]) < TOL_CURVE
    assert np.allclose(b["N"], a["N"], rtol=TOL_CURVE, atol=1e-6 * max(float(np.max(a["N"])), 1e-300))
