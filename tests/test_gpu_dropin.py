"""The drop-in surface beyond apply / J v, through the C ABI, vs the reference's own outputs.

Reference entry points (fixtures from tests/golden/make_golden.py): ``A_lin``
(fvm/operator.py:221), ``jacobian`` as CSR (operator.py:458-471), ``strip_face_currents``
(operator.py:391-399), ``sub_operator`` / ``SubOperatorView`` / ``RestrictedSubOperator``
(operator.py:476-646), ``newton_solve`` iterates, residual norms and ``source``
(newton.py:86-168), ``step`` feeding observers' ``on_iterates`` (timestepping.py:98-101).
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import assert_newton_solution, golden_cases, load_golden, oracle_params, scaled_err
from oracle import fvm_oracle as O

pytestmark = pytest.mark.gpu


def _P():
    import paper_1704_04139_b200 as P
    return P


@pytest.fixture(scope="module", params=golden_cases())
def case(request):
    P = _P()
    g = load_golden(request.param)
    soc, i00pl = g["params"]
    params = P.MaterialParams(soc_init=float(soc), i00_plel=float(i00pl))
    dof = P.build_dofmap(P.PhaseGrid(g["labels"], float(g["voxel_size"])))
    return g, P.SystemOperator(dof, params), dof, params


def test_A_lin_matches_reference(case):
    g, op, dof, _ = case
    A = op.A_lin
    assert isinstance(A, sp.csr_matrix) and A.shape == (dof.n_total, dof.n_total)
    A = A.copy()
    A.sort_indices()
    assert np.array_equal(A.indptr, g["a_indptr"]) and np.array_equal(A.indices, g["a_indices"])
    assert np.max(np.abs(A.data - g["a_data"]) / np.abs(g["a_data"])) < 1e-13


def test_jacobian_is_a_reference_csr(case):
    """jacobian() is a scipy CSR with the reference's pattern and supports the reference's
    own use, ``op.jacobian(...) + sp.diags(mass)`` (newton.py:126)."""
    g, op, dof, _ = case
    x, n_pl, beta = g["x"], g["n_pl"], float(g["beta"])
    J = op.jacobian(x, n_pl, float(g["mu"]), beta=beta)
    assert isinstance(J, sp.csr_matrix)
    J.sort_indices()
    assert np.array_equal(J.indptr, g["j_indptr"]) and np.array_equal(J.indices, g["j_indices"])
    assert scaled_err(J @ g["v"], g["jv"], abs(J) @ np.abs(g["v"])) < 1e-10
    mass = np.zeros(dof.n_total)
    mass[: dof.n_c] = 1.0 / float(g["dt"])
    Jm = (J + sp.diags(mass)).tocsc()
    assert Jm.shape == J.shape
    # the matrix-free operator applies the same matrix on the device
    v = g["v"]
    jop = op.jacobian_operator(x, n_pl, beta=beta, inv_dt=1.0 / float(g["dt"]))
    assert scaled_err(jop @ v, Jm @ v, abs(Jm) @ np.abs(v)) < 1e-10


def test_strip_face_currents_match_reference(case):
    g, op, *_ = case
    cur, slot = op.strip_face_currents(g["x"], g["n_pl"], beta=float(g["beta"]))
    assert np.array_equal(slot, g["strip_slot"])
    ref = g["strip_current"]
    assert np.max(np.abs(cur - ref) / np.maximum(np.abs(ref), 1e-300)) < 1e-10


@pytest.mark.parametrize("which", ["bv", "one_over_c"])
def test_restricted_sub_operator_matches_reference(case, which):
    """Restricted rows + local Jacobian from the stencil values only (the EI access path;
    the same face table and device face kinetics as the ROM online kernel)."""
    g, op, *_ = case
    view = op.sub_operator(which)
    assert view.dim == op.dof.n_total
    assert np.array_equal(view.output_dofs(), g[f"sub_{which}_output_dofs"])
    rs = view.restricted(g[f"sub_{which}_rows"])
    assert np.array_equal(rs.rows, g[f"sub_{which}_rows"])
    assert np.array_equal(rs.stencil, g[f"sub_{which}_stencil"])
    xs = g["x"][rs.stencil]
    beta = float(g["beta"])
    ref = g[f"sub_{which}_apply"]
    Jref = g[f"sub_{which}_jac"]
    got = rs.apply(xs, g["n_pl"], beta=beta)
    scale = np.abs(Jref) @ np.abs(xs) + np.abs(ref)
    assert scaled_err(got, ref, scale) < 1e-10
    Jg = rs.jacobian(xs, g["n_pl"], beta=beta).toarray()
    assert np.max(np.abs(Jg - Jref)) <= 1e-10 * max(np.max(np.abs(Jref)), 1e-300)
    # and the full view agrees with the restricted one at the selected rows
    full = view.apply(g["x"], g["n_pl"], beta=beta)
    assert scaled_err(full[rs.rows], got, scale) < 1e-10


def test_newton_iterates_and_norms_match_reference(case):
    g, op, dof, _ = case
    P = _P()
    x, n_pl = g["x"], g["n_pl"]
    res = P.newton_solve(op, x, float(g["dt"]), x, n_pl, float(g["mu"]), P.SolverConfig())
    ref_its = g["newton_iterates"]
    assert res.n_iter == int(g["newton_iters"]) == len(res.iterates) == ref_its.shape[0]
    nc = dof.n_c
    # intermediate iterates carry the Krylov solve's error of their Newton step (the
    # reference factorizes), amplified by the positivity guard (its step length is set by
    # the single limiting voxel): each agrees with the reference's to 1e-2 of its own step;
    # the converged one to the curve bar (assert_newton_solution)
    prev = x
    for a, b in zip(res.iterates, ref_its):
        step_c, step_p = np.max(np.abs(b[:nc] - prev[:nc])), np.max(np.abs(b[nc:] - prev[nc:]))
        assert np.max(np.abs(a[:nc] - b[:nc])) <= 1e-2 * step_c + 1e-8 * np.max(np.abs(b[:nc]))
        assert np.max(np.abs(a[nc:] - b[nc:])) <= 1e-2 * step_p + 1e-8
        prev = b
    assert_newton_solution(res.iterates[-1], ref_its[-1], nc)
    assert np.array_equal(res.iterates[-1], res.x)
    norms = g["newton_norms"]
    assert len(res.residual_norms) == len(norms)
    assert res.residual_norms[0] == pytest.approx(norms[0], rel=1e-12)
    # later norms sit near the tolerance: same ordering, all decreasing like the reference's
    assert all(b <= a for a, b in zip(res.residual_norms, res.residual_norms[1:]))


def test_newton_source_term_matches_reference(case):
    g, op, dof, _ = case
    P = _P()
    x, n_pl = g["x"], g["n_pl"]
    res = P.newton_solve(op, x, float(g["dt"]), x, n_pl, float(g["mu"]), P.SolverConfig(),
                         source=g["source"])
    orc = O.OracleOperator(g["labels"], float(g["voxel_size"]), oracle_params(g))
    assert_newton_solution(res.x, g["source_x"], dof.n_c, orc, x, n_pl, float(g["mu"]), float(g["dt"]),
                           float(g["beta"]), source=g["source"])
    # and the source changed the solution by far more than the agreement bar
    assert np.max(np.abs(res.x - g["newton_x"])) > 1e3 * np.max(np.abs(res.x - g["source_x"]))


class _Recorder:
    def __init__(self):
        self.iterates, self.states = [], []

    def on_iterates(self, iterates, n_pl, mu, t):
        self.iterates.append((len(iterates), iterates[-1].copy() if len(iterates) else None, t))

    def on_state(self, state, op, mu):
        self.states.append(state.t)


def test_step_feeds_observers_and_run_transient_call_pattern(case):
    """The reference's run_transient / step call pattern with observers (timestepping.py:
    64-106, 117-176): on_iterates receives the accepted solve's iterates, whose last one is
    the new state; on_state sees every recorded state."""
    g, op, dof, params = case
    P = _P()
    mu, dt = float(g["mu"]), float(g["dt"])
    cfg = P.SolverConfig(dt_init=dt, dt_max=dt)
    rec = _Recorder()
    traj = P.run_transient(dof.grid, params, P.BoundaryDrive(mu), cfg, 3 * dt, observers=(rec,), op=op)
    assert len(rec.states) == len(traj.states) == 4
    assert len(rec.iterates) == 3
    for (k, last, t), n_it, st in zip(rec.iterates, traj.newton_iters, traj.states[1:]):
        assert k == n_it >= 1
        assert t == pytest.approx(st.t)
        assert np.array_equal(last, st.x)
    v_cp, _ = P.qoi_vectors(dof)
    assert np.max(np.abs(np.array([v_cp @ s.x for s in traj.states]) - g["traj_voltage"][:4])
                  / np.abs(g["traj_voltage"][:4])) < 1e-6


def test_device_resident_state_steps_like_host_state(case):
    """A CellState holding CUDA tensors steps on the device with the same result."""
    g, op, dof, params = case
    P = _P()
    mu, dt = float(g["mu"]), float(g["dt"])
    cfg = P.SolverConfig()
    s0 = P.prepare_initial_state(op, params, mu, cfg)
    a, *_ = P.step(op, s0, dt, mu, cfg)
    b, *_ = P.step(op, s0.to_device(), dt, mu, cfg)
    assert not isinstance(b.c, np.ndarray)
    hb = b.to_host()
    # same operator, same solver path: at most the preconditioner refresh differs
    assert np.allclose(hb.c, a.c, rtol=1e-9, atol=0) and np.allclose(hb.phi, a.phi, rtol=0, atol=1e-9)
    assert np.allclose(hb.n_pl, a.n_pl, rtol=1e-9, atol=0)
    assert P.qoi_cell_voltage(b, dof) == pytest.approx(P.qoi_cell_voltage(a, dof), rel=1e-9)


def test_system_operator_takes_over_the_dofmap_geometry():
    """``SystemOperator(dofmap, params)`` re-parametrises the device geometry that
    ``build_dofmap`` classified (``hc_operator_set_params``) instead of classifying the grid
    twice; it must equal an operator built from scratch with those parameters, bit for bit,
    after work that depends on the parameters (multigrid, solver graphs) has run."""
    P = _P()
    g = load_golden(golden_cases()[0])
    soc, i00pl = g["params"]
    params = P.MaterialParams(soc_init=float(soc), i00_plel=float(i00pl), kappa_el=0.8, i00_grel=3.0e-4)
    grid = P.PhaseGrid(g["labels"], float(g["voxel_size"]))
    dof = P.build_dofmap(grid)
    assert dof._nat is not None
    handed = P.SystemOperator(dof, params)      # takes the Dofmap's device operator
    assert dof._nat is None
    fresh = P.SystemOperator(dof, params)       # nothing left to take: classifies again
    assert handed.native is not fresh.native
    x, n_pl, mu, beta, v, dt = g["x"], g["n_pl"], float(g["mu"]), float(g["beta"]), g["v"], float(g["dt"])
    assert handed.n_const == fresh.n_const and handed.gX == fresh.gX
    assert np.array_equal(handed.apply(x, n_pl, mu, beta=beta), fresh.apply(x, n_pl, mu, beta=beta))
    assert np.array_equal(handed.jvp(x, n_pl, v, beta=beta), fresh.jvp(x, n_pl, v, beta=beta))
    cfg = P.SolverConfig()
    a = P.newton_solve(handed, x, dt, x, n_pl, mu, cfg)
    b = P.newton_solve(fresh, x, dt, x, n_pl, mu, cfg)
    assert a.n_iter == b.n_iter and a.krylov_iters == b.krylov_iters
    assert np.array_equal(a.x, b.x)
