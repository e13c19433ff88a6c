"""GPU: size-independent properties at the BASELINE config sizes (tiny / medium cells):
J v linearity and agreement with central differences of the residual, lithium
conservation of an implicit step, bit-reproducible index work and idempotent setup."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cell(name):
    import paper_1704_04139_b200 as P
    from paper_1704_04139_b200.configs import CONFIGS
    from paper_1704_04139_b200.microgen import generate_cell
    rs = CONFIGS[name]
    grid = generate_cell(rs.cell)
    params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
    op = P.SystemOperator(P.build_dofmap(grid), params)
    h = grid.voxel_size * 1e-6
    mu = -rs.c_rate * params.c_gr_max * params.constants.F * np.count_nonzero(grid.labels == 1) \
        * h ** 3 / 3600 / (grid.labels.shape[1] * grid.labels.shape[2] * h * h)
    return P, rs, grid, params, op, mu


@pytest.mark.parametrize("name", ["tiny", "medium"])
def test_jvp_linear_and_matches_central_differences(name):
    P, rs, grid, params, op, mu = _cell(name)
    st = P.initial_fields(op.dof, params)
    rng = np.random.default_rng(1)
    x = st.x.copy()
    x[: op.dof.n_c] *= 1.0 + 0.02 * rng.standard_normal(op.dof.n_c)
    x[op.dof.n_c:] += 0.005 * rng.standard_normal(op.dof.n_p)
    beta = rs.dt * op.face_area / params.constants.F
    v, w = rng.standard_normal(op.dof.n_total), rng.standard_normal(op.dof.n_total)
    v[: op.dof.n_c] *= 1e-3 * np.abs(x[: op.dof.n_c])   # relative perturbations of c
    w[: op.dof.n_c] *= 1e-3 * np.abs(x[: op.dof.n_c])
    v[op.dof.n_c:] *= 1e-4
    w[op.dof.n_c:] *= 1e-4
    jv, jw = op.jvp(x, st.n_pl, v, beta=beta), op.jvp(x, st.n_pl, w, beta=beta)
    jvw = op.jvp(x, st.n_pl, 2.0 * v - 3.0 * w, beta=beta)
    assert np.max(np.abs(jvw - (2.0 * jv - 3.0 * jw))) <= 1e-9 * np.max(np.abs(jvw))
    eps = 1e-4
    fp = op.apply(x + eps * v, st.n_pl, mu, beta=beta)
    fm = op.apply(x - eps * v, st.n_pl, mu, beta=beta)
    fd = (fp - fm) / (2 * eps)
    assert np.linalg.norm(fd - jv) <= 1e-5 * np.linalg.norm(jv)


@pytest.mark.parametrize("name", ["tiny", "medium"])
def test_step_conserves_lithium(name):
    """An implicit step moves lithium only through the counter-electrode faces:
    d(sum c V + sum n_pl) = dt * sum_CE i A / F at the new state (to solver tolerance)."""
    P, rs, grid, params, op, mu = _cell(name)
    cfg = P.SolverConfig(dt_init=min(0.05, rs.dt), dt_max=rs.dt)
    st0 = P.prepare_initial_state(op, params, mu, cfg)
    st1, dt, _, info = P.step(op, st0, rs.dt, mu, cfg)
    V = op.voxel_volume
    li0 = st0.c.sum() * V + st0.n_pl.sum()
    li1 = st1.c.sum() * V + st1.n_pl.sum()
    # counter-electrode current at the new state: exchange current on foil|electrolyte faces
    x = st1.x
    vt = params.thermal_voltage_2
    i_ce = 2.0 * params.i00_ceel * np.sinh((x[op.ce_xp_fo] - x[op.ce_xp_el]) / vt)
    # positive (anodic) foil current dissolves the foil: lithium enters the electrolyte
    flux_in = (i_ce * op.face_area / params.constants.F).sum()
    assert abs((li1 - li0) - dt * flux_in) <= 1e-6 * abs(dt * flux_in) + 1e-12 * abs(li0)
    assert st1.n_pl.min() >= 0.0


def test_setup_is_reproducible():
    P, rs, grid, params, op, mu = _cell("tiny")
    d2 = P.build_dofmap(grid)
    op2 = P.SystemOperator(d2, params)
    assert np.array_equal(op.dof.c_dof, d2.c_dof) and np.array_equal(op.dof.p_dof, d2.p_dof)
    for a in ("bv_xc_gr", "ce_xp_fo", "strip_xp_pl", "strip_slot", "elel_xc_i"):
        assert np.array_equal(getattr(op, a), getattr(op2, a))


def test_steps_are_bitwise_reproducible():
    """No floating-point atomics and fixed-order reductions on the solver path (parallel
    preconditioner branches, fused J v partials, last-block finishes): two runs from fresh
    operators give bitwise identical states."""
    P, rs, grid, params, _, mu = _cell("tiny")
    out = []
    for _ in range(2):
        op = P.SystemOperator(P.build_dofmap(grid), params)
        cfg = P.SolverConfig(dt_init=min(0.05, rs.dt), dt_max=rs.dt, linear_safety=0.3)
        st = P.prepare_initial_state(op, params, mu, cfg)
        for _ in range(3):
            st, _, _, _ = P.step(op, st, rs.dt, mu, cfg)
        out.append((st.x.copy(), st.n_pl.copy()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_ragged_grid_is_bitwise_reproducible():
    """The cp.async stencil path (x pitch without tensor-map tiles: the 10x10x20 reference
    fixture) gathers its interface currents per voxel in direction order — no atomics —
    so residuals and steps from fresh operators are bitwise identical."""
    from conftest import load_golden
    import paper_1704_04139_b200 as P
    g = load_golden("refgen_10x10x20")
    soc, i00pl = g["params"]
    params = P.MaterialParams(soc_init=float(soc), i00_plel=float(i00pl))
    grid = P.PhaseGrid(g["labels"], float(g["voxel_size"]))
    x, n_pl, mu, beta, dt = g["x"], g["n_pl"], float(g["mu"]), float(g["beta"]), float(g["dt"])
    out = []
    for _ in range(2):
        op = P.SystemOperator(P.build_dofmap(grid), params)
        r = op.apply(x, n_pl, mu, beta=beta)
        cfg = P.SolverConfig()
        st = P.prepare_initial_state(op, params, mu, cfg)
        for _ in range(2):
            st, _, _, _ = P.step(op, st, dt, mu, cfg)
        out.append((r, st.x.copy(), st.n_pl.copy()))
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("safety", [0.1, 0.3])
def test_inexact_newton_curves_match_exact_on_tiny_config(safety):
    """BASELINE config 0 (tiny cell, 1C, dt = 1 s, 10 steps): the voltage, mean solid
    concentration and plated-inventory curves with an inexact-Newton Krylov tolerance
    (linear_safety: Krylov stops at safety x the Newton tolerance) agree with the
    exact-tolerance path within 1e-6."""
    P, rs, grid, params, op, mu = _cell("tiny")
    v_cp, v_ac = P.qoi_vectors(op.dof)
    curves = {}
    for ls in (0.0, safety):
        cfg = P.SolverConfig(dt_init=min(0.05, rs.dt), dt_max=rs.dt, linear_safety=ls)
        st = P.prepare_initial_state(op, params, mu, cfg)
        vs, cs, ns = [], [], []
        for _ in range(rs.n_steps):
            st, _, _, _ = P.step(op, st, rs.dt, mu, cfg)
            vs.append(v_cp @ st.x)
            cs.append(v_ac @ st.x)
            ns.append(st.n_pl.sum())
        curves[ls] = (np.array(vs), np.array(cs), np.array(ns))
    (v0, c0, n0), (v1, c1, n1) = curves[0.0], curves[safety]
    assert np.max(np.abs(v1 - v0) / np.abs(v0)) < 1e-6
    assert np.max(np.abs(c1 - c0) / np.abs(c0)) < 1e-6
    assert np.allclose(n1, n0, rtol=1e-6, atol=0.0)
