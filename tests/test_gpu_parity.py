"""GPU parity: the CUDA path through the C ABI vs reference fixtures and the CPU oracle.

Bars: index work bit-exact; residual and J v within 1e-10 relative (per row,
relative to the sum of |contributions|); voltage / plated-lithium curves within
1e-6 relative.
"""

import numpy as np
import pytest

from conftest import assert_newton_solution, golden_cases, load_golden, oracle_params, scaled_err
from oracle import fvm_oracle as O

pytestmark = pytest.mark.gpu

TOL_RES = 1e-10


def _pkg():
    import paper_1704_04139_b200 as P
    from paper_1704_04139_b200 import params as prm
    return P, prm


def _gpu_op(g):
    P, prm = _pkg()
    soc, i00pl = g["params"]
    params = P.MaterialParams(soc_init=float(soc), i00_plel=float(i00pl))
    grid = P.PhaseGrid(g["labels"], float(g["voxel_size"]))
    dof = P.build_dofmap(grid)
    return P.SystemOperator(dof, params), dof, params


@pytest.fixture(scope="module", params=golden_cases())
def case(request):
    g = load_golden(request.param)
    op, dof, params = _gpu_op(g)
    orc = O.OracleOperator(g["labels"], float(g["voxel_size"]), oracle_params(g))
    return g, op, dof, params, orc


def test_dofmap_bit_exact(case):
    g, op, dof, _, _ = case
    assert np.array_equal(dof.c_dof, g["c_dof"])
    assert np.array_equal(dof.p_dof, g["p_dof"])
    assert np.array_equal(dof.plated_voxels, g["plated"])
    assert np.array_equal(dof.dirichlet, g["dirichlet"])


def test_face_lists_bit_exact(case):
    g, op, *_ = case
    assert np.array_equal(np.stack([op.bv_xc_gr, op.bv_xc_el, op.bv_xp_gr, op.bv_xp_el]), g["bv"])
    assert np.array_equal(np.stack([op.ce_xp_fo, op.ce_xc_el, op.ce_xp_el]), g["ce"])
    assert np.array_equal(np.stack([op.strip_xp_pl, op.strip_xc_el, op.strip_xp_el,
                                    op.strip_slot]), g["strip"])
    assert np.array_equal(np.stack([op.elel_xc_i, op.elel_xc_j, op.elel_xp_i, op.elel_xp_j]),
                          g["elel"])


def test_residual_parts(case):
    g, op, dof, _, orc = case
    x, n_pl, mu, beta = g["x"], g["n_pl"], float(g["mu"]), float(g["beta"])
    scale = orc.row_scale(x, n_pl, mu, beta)
    assert scaled_err(op.apply(x, n_pl, mu, beta=beta), g["apply"], scale) < TOL_RES
    assert scaled_err(op.apply_bv(x, n_pl, beta=beta), g["apply_bv"], scale) < TOL_RES
    assert scaled_err(op.apply_one_over_c(x), g["apply_1c"], scale) < TOL_RES
    assert scaled_err(op.apply_lin(x), g["apply_lin"], scale) < TOL_RES
    assert np.array_equal(op.b_bnd, g["b_bnd"])


def test_jvp(case):
    g, op, dof, _, orc = case
    x, n_pl, beta, v = g["x"], g["n_pl"], float(g["beta"]), g["v"]
    Jo = orc.jacobian(x, n_pl, beta)
    scale = abs(Jo) @ np.abs(v)
    assert scaled_err(op.jvp(x, n_pl, v, beta=beta), g["jv"], scale) < TOL_RES
    # mass term on the c block
    jm = op.jvp(x, n_pl, v, beta=beta, inv_dt=2.0)
    ref = g["jv"].copy()
    ref[: dof.n_c] += 2.0 * v[: dof.n_c]
    assert scaled_err(jm, ref, scale + 2.0 * np.abs(np.r_[v[: dof.n_c], 0 * v[dof.n_c:]])) < TOL_RES


def test_jacobian_sparsity_bit_exact(case):
    g, op, *_ = case
    J = op.jacobian(g["x"], g["n_pl"], beta=float(g["beta"])).tocsr()
    J.sort_indices()
    assert np.array_equal(J.indptr, g["j_indptr"])
    assert np.array_equal(J.indices, g["j_indices"])


def test_newton_solve(case):
    g, op, dof, _, _ = case
    P, _ = _pkg()
    x, n_pl = g["x"], g["n_pl"]
    res = P.newton_solve(op, x, float(g["dt"]), x, n_pl, float(g["mu"]), P.SolverConfig())
    orc = case[4]
    assert_newton_solution(res.x, g["newton_x"], dof.n_c, orc, x, n_pl, float(g["mu"]), float(g["dt"]),
                           float(g["beta"]))


@pytest.mark.parametrize("linear_safety", [0.0, 0.1, 0.3])
def test_transient_curves(case, linear_safety):
    """Curves vs the reference; also with the inexact-Newton Krylov tolerance the bench
    uses (linear_safety=0.1: never solve beyond what the Newton tolerance can use)."""
    g, op, dof, params, _ = case
    P, _ = _pkg()
    mu, dt = float(g["mu"]), float(g["dt"])
    cfg = P.SolverConfig(linear_safety=linear_safety)
    state = P.prepare_initial_state(op, params, mu, cfg)
    v_cp, v_ac = P.qoi_vectors(dof)
    volts, means, npls = [v_cp @ state.x], [v_ac @ state.x], [state.n_pl.sum()]
    for _ in range(4):
        state, dt_used, _, info = P.step(op, state, dt, mu, cfg)
        assert dt_used == pytest.approx(dt) and info.retries == 0
        volts.append(v_cp @ state.x)
        means.append(v_ac @ state.x)
        npls.append(state.n_pl.sum())
    assert np.max(np.abs(np.array(volts) - g["traj_voltage"]) / np.abs(g["traj_voltage"])) < 1e-6
    assert np.max(np.abs(np.array(means) - g["traj_mean_c"]) / np.abs(g["traj_mean_c"])) < 1e-6
    assert np.allclose(npls, g["traj_npl"], rtol=1e-6, atol=1e-24)


def test_model_errors_match_reference():
    P, _ = _pkg()
    lab = np.zeros((6, 4, 4), dtype=np.uint8)
    lab[-1] = P.Phase.COLLECTOR_COUNTER
    with pytest.raises(P.ModelError, match="no graphite"):
        P.build_dofmap(P.PhaseGrid(lab, 1.0))
    lab[1] = P.Phase.GRAPHITE
    with pytest.raises(P.ModelError, match="lithium foil"):
        P.build_dofmap(P.PhaseGrid(lab, 1.0))
    lab[4] = P.Phase.LI_FOIL
    lab[2, 0, 0] = P.Phase.LI_FOIL      # foil touching graphite: forbidden
    with pytest.raises(P.ModelError, match="forbidden"):
        P.build_dofmap(P.PhaseGrid(lab, 1.0))
    lab[2, 0, 0] = P.Phase.ELECTROLYTE
    lab[2:4] = P.Phase.COLLECTOR_WORKING  # no electrolyte path
    with pytest.raises(P.ModelError, match="electrolyte path"):
        P.build_dofmap(P.PhaseGrid(lab, 1.0))


def test_tiny_config_residual_vs_oracle():
    """BASELINE config 0 geometry (32x32x64): residual + J v vs the oracle."""
    P, _ = _pkg()
    from paper_1704_04139_b200.configs import CONFIGS
    from paper_1704_04139_b200.microgen import generate_cell
    grid = generate_cell(CONFIGS["tiny"].cell)
    params = P.MaterialParams(soc_init=0.1, i00_plel=1e-3 / np.sqrt(1000.0))
    op = P.SystemOperator(P.build_dofmap(grid), params)
    orc = O.OracleOperator(grid.labels, grid.voxel_size, O.Params(soc_init=0.1,
                                                                    i00_plel=1e-3 / np.sqrt(1000.0)))
    rng = np.random.default_rng(5)
    x, n_pl = O.initial_fields(orc)
    x[: orc.n_c] *= 1.0 + 0.05 * rng.standard_normal(orc.n_c)
    x[orc.n_c:] += 0.01 * rng.standard_normal(orc.n_p)
    beta = 0.5 * orc.face_area / orc.p.F
    r_ref = orc.apply(x, n_pl, -10.0, beta)
    assert scaled_err(op.apply(x, n_pl, -10.0, beta=beta), r_ref,
                      orc.row_scale(x, n_pl, -10.0, beta)) < TOL_RES
    v = rng.standard_normal(orc.n)
    J = orc.jacobian(x, n_pl, beta)
    assert scaled_err(op.jvp(x, n_pl, v, beta=beta), J @ v, abs(J) @ np.abs(v)) < TOL_RES
