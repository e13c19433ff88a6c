"""GPU: reduced-order model (BASELINE config 4 pipeline) — offline build on the device,
online loop in one kernel, checked against the CPU restatement (oracle/rom_oracle.py)
and against the full-order trajectory it was trained on."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_TRAIN = 12


@pytest.fixture(scope="module")
def cell():
    import paper_1704_04139_b200 as P
    from paper_1704_04139_b200 import mor
    from paper_1704_04139_b200.microgen import CellSpec, generate_cell
    from oracle import fvm_oracle as O
    spec = CellSpec(16, 16, 32, 14, 4, seed=7, radius_mean=3.0, porosity=0.35, plating_intensity=0.05)
    grid = generate_cell(spec)
    params = P.MaterialParams()
    op = P.SystemOperator(P.build_dofmap(grid), params)
    h = grid.voxel_size * 1e-6
    mu = -2.0 * params.c_gr_max * params.constants.F * np.count_nonzero(grid.labels == 1) * h ** 3 \
        / 3600.0 / (grid.labels.shape[1] * grid.labels.shape[2] * h * h)
    dt = 1.0
    cfg = P.SolverConfig(dt_init=dt, dt_max=dt)
    st = P.prepare_initial_state(op, params, mu, cfg)
    snaps = mor.collect_snapshots(op, st.x, st.n_pl, mu, dt, N_TRAIN)
    orc = O.OracleOperator(grid.labels, grid.voxel_size, O.Params())
    return dict(op=op, orc=orc, st=st, mu=mu, dt=dt, snaps=snaps)


def _rom(cell, k, m):
    from paper_1704_04139_b200 import mor
    return mor.build_rom(cell["op"], cell["snaps"], k, k, m)


def test_pod_rank_orthonormal(cell):
    from paper_1704_04139_b200 import mor
    X = cell["snaps"].X
    V, sig = mor.pod_rank(X[: cell["op"].dof.n_c], 6)
    G = (V.t() @ V).cpu().numpy()
    assert np.max(np.abs(G - np.eye(G.shape[0]))) < 1e-12
    ref = np.linalg.svd(X[: cell["op"].dof.n_c].cpu().numpy(), compute_uv=False)
    assert np.allclose(sig.cpu().numpy()[:4], ref[:4], rtol=1e-8)


def test_deim_blocked_equals_sequential_greedy():
    from paper_1704_04139_b200 import mor
    from oracle import rom_oracle as R
    rng = np.random.default_rng(5)
    W = rng.standard_normal((3000, 37)) * 10.0 ** -(0.1 * np.arange(37))
    assert np.array_equal(mor.deim(W, block=8), R.deim(W))


def test_ei_exact_at_interpolation_rows(cell):
    import torch
    rom = _rom(cell, 6, 10)
    snaps = cell["snaps"]
    W, pi = rom.W, torch.as_tensor(rom.pi, device="cuda")
    for s in (0, N_TRAIN // 2, N_TRAIN):
        Nx = snaps.N[:, s]
        coef = torch.linalg.solve(W[pi], Nx[pi])
        interp = W @ coef
        assert torch.max(torch.abs(interp[pi] - Nx[pi])) <= 1e-12 * torch.max(torch.abs(Nx[pi]))


def test_rom_online_matches_cpu_restatement(cell):
    from paper_1704_04139_b200 import mor
    from oracle import rom_oracle as R
    rom = _rom(cell, 6, 10)
    xt0 = rom.project(cell["st"].x)
    npl0 = cell["st"].n_pl
    n = 6
    tr = mor.solve_rom(cell["op"], rom, xt0, npl0, cell["mu"], cell["dt"], n)
    xo, no, qo, io = R.rom_run(cell["orc"], rom.host(), xt0.cpu().numpy(), npl0, cell["mu"], cell["dt"], n)
    assert np.array_equal(tr.newton_iters, io)
    xg = tr.xt.cpu().numpy()
    k_c = rom.k_c
    assert np.max(np.abs(xg[:k_c] - xo[:k_c])) <= 1e-10 * np.max(np.abs(xo[:k_c]))
    assert np.max(np.abs(xg[k_c:] - xo[k_c:])) <= 1e-10 * (np.max(np.abs(xo[k_c:])) + 1.0)
    assert np.allclose(tr.voltage, qo[:, 0], rtol=1e-10, atol=1e-12)
    assert np.allclose(tr.mean_solid_c, qo[:, 1], rtol=1e-10)
    if npl0.size:
        assert np.allclose(tr.n_pl.cpu().numpy()[: npl0.size], no, rtol=1e-10, atol=1e-30)


def test_rom_reproduces_training_trajectory(cell):
    """Training parameter: ROM QoI curves follow the full-order ones (SPEC mor: max
    relative QoI deviation <= 1e-3)."""
    from paper_1704_04139_b200 import mor
    from paper_1704_04139_b200.qoi import qoi_vectors
    op, snaps = cell["op"], cell["snaps"]
    rom = _rom(cell, 10, 24)
    tr = mor.solve_rom(op, rom, rom.project(cell["st"].x), cell["st"].n_pl, cell["mu"], cell["dt"], N_TRAIN)
    v_cp, v_ac = qoi_vectors(op.dof)
    X = snaps.X.cpu().numpy()
    fom_v, fom_ac = v_cp @ X[:, 1:], v_ac @ X[:, 1:]
    assert np.max(np.abs(tr.voltage - fom_v)) <= 1e-3 * np.max(np.abs(fom_v))
    assert np.max(np.abs(tr.mean_solid_c - fom_ac) / np.abs(fom_ac)) <= 1e-3


def test_error_estimator_twin_and_true_error(cell):
    """SPEC mor.estimate_error: twin = same model -> 0; otherwise the estimate tracks the
    true ROM error (vs the full-order trajectory) within a factor 10."""
    import torch
    from paper_1704_04139_b200 import mor
    op, snaps, st = cell["op"], cell["snaps"], cell["st"]
    rom, twin = mor.build_rom_twin(op, snaps, 8, 8, 16, keep_fraction=0.75)
    ec, ep = mor.estimate_error(op, twin, twin, st.x, st.n_pl, cell["mu"], cell["dt"], N_TRAIN)
    assert ec == 0.0 and ep == 0.0
    ec, ep = mor.estimate_error(op, rom, twin, st.x, st.n_pl, cell["mu"], cell["dt"], N_TRAIN)
    assert ec > 0.0 and ep > 0.0
    tr = mor.solve_rom(op, rom, rom.project(st.x), st.n_pl, cell["mu"], cell["dt"], N_TRAIN, keep_states=True)
    nc = op.dof.n_c
    X = snaps.X[:, 1:].t()                         # (steps, n)
    L = torch.stack([rom.lift(tr.states[i]) for i in range(N_TRAIN)])
    true_c = float(torch.max(torch.linalg.vector_norm(L[:, :nc] - X[:, :nc], dim=1)
                             / torch.linalg.vector_norm(X[:, :nc], dim=1)))
    assert 0.1 <= ec / true_c <= 10.0


def test_batched_rom_equals_single_trajectories(cell):
    """One cluster per applied current in one launch = the single-trajectory runs."""
    from paper_1704_04139_b200 import mor
    op, st = cell["op"], cell["st"]
    rom = _rom(cell, 6, 10)
    xt0 = rom.project(st.x)
    mus = [cell["mu"], 0.8 * cell["mu"], 1.1 * cell["mu"]]
    v, c, xt = mor.solve_rom_batch(op, rom, xt0, st.n_pl, mus, cell["dt"], 5)
    for i, mu in enumerate(mus):
        tr = mor.solve_rom(op, rom, xt0, st.n_pl, mu, cell["dt"], 5)
        assert np.allclose(v[i], tr.voltage, rtol=1e-13, atol=1e-15)
        assert np.allclose(c[i], tr.mean_solid_c, rtol=1e-13)
        assert np.allclose(xt[i].cpu().numpy(), tr.xt.cpu().numpy(), rtol=1e-12, atol=1e-12)


def test_separate_ei_spaces_and_tolerance_truncation(cell):
    """SPEC build_rom / pod: A_bv and A_1/c interpolated in their own EI spaces (each row
    reads only its sub-operator's faces), POD ranks from the discarded-energy tolerance;
    the online kernel still equals the CPU restatement and follows the training run."""
    from paper_1704_04139_b200 import mor
    from paper_1704_04139_b200.qoi import qoi_vectors
    from oracle import rom_oracle as R
    op, snaps, st = cell["op"], cell["snaps"], cell["st"]
    Vc, sig = mor.pod_rank(snaps.X[: op.dof.n_c], None, rel_tol=1e-7)
    lam = (sig.cpu().numpy() ** 2)
    k = Vc.shape[1]
    assert lam[k:].sum() <= 1e-14 * lam.sum() and (k == 1 or lam[k - 1:].sum() > 1e-14 * lam.sum())
    rom = mor.build_rom(op, snaps, 10, 10, 12, separate_ei=True, m_c=12)
    assert rom.m == 24 and rom.W is None
    xt0 = rom.project(st.x)
    tr = mor.solve_rom(op, rom, xt0, st.n_pl, cell["mu"], cell["dt"], N_TRAIN)
    xo, no, qo, io = R.rom_run(cell["orc"], rom.host(), xt0.cpu().numpy(), st.n_pl, cell["mu"], cell["dt"], N_TRAIN)
    assert np.array_equal(tr.newton_iters, io)
    assert np.allclose(tr.voltage, qo[:, 0], rtol=1e-10, atol=1e-12)
    v_cp, _ = qoi_vectors(op.dof)
    fom_v = v_cp @ snaps.X.cpu().numpy()[:, 1:]
    assert np.max(np.abs(tr.voltage - fom_v)) <= 1e-3 * np.max(np.abs(fom_v))
