"""Pin the CPU oracle against fixtures produced by the reference implementation."""

import numpy as np
import pytest

from conftest import golden_cases, load_golden, oracle_params, scaled_err
from oracle import fvm_oracle as O


@pytest.fixture(scope="module", params=golden_cases())
def case(request):
    g = load_golden(request.param)
    op = O.OracleOperator(g["labels"], float(g["voxel_size"]), oracle_params(g))
    return g, op


def test_dofmap_bit_exact(case):
    g, op = case
    assert np.array_equal(op.c_dof, g["c_dof"])
    assert np.array_equal(op.p_dof, g["p_dof"])
    assert np.array_equal(op.plated, g["plated"])
    assert np.array_equal(op.dirichlet, g["dirichlet"])


def test_face_lists_bit_exact(case):
    g, op = case
    assert np.array_equal(np.stack(op.bv), g["bv"])
    assert np.array_equal(np.stack(op.ce), g["ce"])
    assert np.array_equal(np.stack(op.strip), g["strip"])
    assert np.array_equal(np.stack(op.elel), g["elel"])


def test_operator_parts(case):
    g, op = case
    x, n_pl, mu, beta = g["x"], g["n_pl"], float(g["mu"]), float(g["beta"])
    scale = op.row_scale(x, n_pl, mu, beta)
    assert scaled_err(op.apply(x, n_pl, mu, beta), g["apply"], scale) < 1e-12
    assert scaled_err(op.apply_bv(x, n_pl, beta), g["apply_bv"], scale) < 1e-12
    assert scaled_err(op.apply_one_over_c(x), g["apply_1c"], scale) < 1e-12
    assert scaled_err(op.apply_lin(x), g["apply_lin"], scale) < 1e-12
    assert np.array_equal(op.b_bnd, g["b_bnd"])


def test_jacobian_pattern_and_product(case):
    g, op = case
    x, n_pl, beta = g["x"], g["n_pl"], float(g["beta"])
    J = op.jacobian(x, n_pl, beta)
    J.sort_indices()
    assert np.array_equal(J.indptr, g["j_indptr"])
    assert np.array_equal(J.indices, g["j_indices"])
    jv = J @ g["v"]
    scale = abs(J) @ np.abs(g["v"])
    assert scaled_err(jv, g["jv"], scale) < 1e-12


def test_newton_matches_reference(case):
    g, op = case
    x, n_pl = g["x"], g["n_pl"]
    xn, it, _ = O.newton_solve(op, x, float(g["dt"]), x, n_pl, float(g["mu"]))
    assert it == int(g["newton_iters"])
    nc = op.n_c
    assert np.max(np.abs(xn[:nc] - g["newton_x"][:nc]) / np.abs(g["newton_x"][:nc])) < 1e-9
    assert np.max(np.abs(xn[nc:] - g["newton_x"][nc:])) < 1e-9


def test_transient_curves_match_reference(case):
    g, op = case
    mu, dt = float(g["mu"]), float(g["dt"])
    x, n_pl = O.initial_fields(op)
    x = O.solve_initial_potential(op, x, n_pl, mu)
    v_cp, v_ac = O.qoi_vectors(op)
    volts, means, npls = [v_cp @ x], [v_ac @ x], [n_pl.sum()]
    for _ in range(4):
        x, n_pl, _, _ = O.step(op, x, n_pl, dt, mu)
        volts.append(v_cp @ x)
        means.append(v_ac @ x)
        npls.append(n_pl.sum())
    assert np.max(np.abs(np.array(volts) - g["traj_voltage"]) / np.abs(g["traj_voltage"])) < 1e-8
    assert np.max(np.abs(np.array(means) - g["traj_mean_c"]) / np.abs(g["traj_mean_c"])) < 1e-10
    assert np.allclose(npls, g["traj_npl"], rtol=1e-8, atol=1e-30)


# Known-answer values frozen in the reference test suite (tests/test_kinetics.py).
# The two marked "frozen parameters" were frozen with i00_ceel = 20 and i00_plel = 0.3,
# which differ from today's MaterialParams defaults (the reference's own tests fail on
# them with the shipped defaults), so they are checked at the parameters they encode.
def test_reference_known_answers():
    p = O.Params()
    assert p.R * p.temperature / 1000.0 == pytest.approx(2.478968175, rel=1e-10)
    flat = O.Params(ocp_table=((0.0, 0.0), (1.0, 0.0)), i00_grel=1.0)
    op = O.OracleOperator.__new__(O.OracleOperator)
    op.p = flat
    assert op._bv(np.array([1.0]), np.array([1.0]), np.array([0.05]), np.array([0.0]))[0] == \
        pytest.approx(2.2680412666023585, rel=1e-12)
    op.p = O.Params(i00_ceel=20.0)        # frozen parameters
    assert op._ce(np.array([0.03]), np.array([0.0]))[0] == pytest.approx(24.702376156555641, rel=1e-12)
    op.p = O.Params(i00_plel=0.3)         # frozen parameters
    op.n_const = 5.0e-15
    i = op._strip(np.array([1000.0]), np.array([0.01]), np.array([0.0]), np.array([5.0e-15]))
    assert i[0] == pytest.approx(-2.0466908437888227, rel=1e-12)
    assert O.f_pre(3.7e-15, 3.7e-15) == pytest.approx(0.5, rel=1e-15)
    assert O.f_pre(2 * 3.7e-15, 3.7e-15) == pytest.approx(16.0 / 17.0, rel=1e-15)


def test_ocp_table_semantics():
    p = O.Params()
    for s, v in p.ocp_table:
        assert p.ocp(s * p.c_gr_max) == pytest.approx(v)
    assert p.ocp(1.5 * p.c_gr_max) == p.ocp_table[-1][1]
    assert p.ocp(0.0) == p.ocp_table[0][1]
