"""GPU: batched stepping equals single-cell stepping; POD Gram on DMMA vs fp64 reference."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_batch_step_matches_single_cell_steps():
    import torch
    import paper_1704_04139_b200 as P
    from paper_1704_04139_b200 import batch as B
    from paper_1704_04139_b200.microgen import CellSpec
    spec = CellSpec(16, 16, 32, 14, 4, seed=100, radius_mean=3.0, porosity=0.35, plating_intensity=0.05)
    cfg = P.SolverConfig(dt_init=0.5, dt_max=0.5)
    cells = B.make_batch(3, first_seed=100, spec=spec, cfg=cfg)
    singles = []
    for c in cells:
        st = P.CellState.from_x(c.x.cpu().numpy(), c.op.dof.n_c, c.n_pl.cpu().numpy()[: c.op.dof.n_plated], 0.0)
        for _ in range(2):
            st, _, _, _ = P.step(c.op, st, 0.5, c.mu, cfg)
        singles.append(st.x)
    for _ in range(2):
        B.step_batch(cells, 0.5, cfg, n_threads=3)
    for c, xs in zip(cells, singles):
        # same kernels; the residual's interface-face atomics make the last bits
        # order dependent, so agreement is at Newton-tolerance level
        nc = c.op.dof.n_c
        xb = c.x.cpu().numpy()
        assert np.max(np.abs(xb[:nc] - xs[:nc]) / np.abs(xs[:nc])) < 1e-9
        assert np.max(np.abs(xb[nc:] - xs[nc:])) < 1e-9


def test_pod_gram_matches_fp64_reference():
    import torch
    from paper_1704_04139_b200 import pod
    rng = np.random.default_rng(3)
    # partial edge tiles (7, 130, 80, 153, 400 snapshots on 64 x 64 tiles); odd counts exercise
    # the half-filled 16-byte column pairs at the edge of a staged panel
    for n_dof, n_snap in ((1000, 7), (50_000, 130), (3_000, 80), (2_500, 153), (4_000, 400)):
        S = rng.standard_normal((n_dof, n_snap))
        w = rng.uniform(0.5, 1.5, n_dof)
        G = pod.pod_gram(S, w)
        ref = (S.T * w) @ S
        assert np.max(np.abs(G - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_pod_basis_orthonormal_and_singular_values():
    from paper_1704_04139_b200 import pod
    rng = np.random.default_rng(4)
    S = rng.standard_normal((50, 8)) @ np.diag(10.0 ** -(0.4 * np.arange(8)))
    B, sig = pod.pod_basis(S, 1e-12)
    assert np.max(np.abs(B.T @ B - np.eye(B.shape[1]))) < 1e-12
    ref = np.linalg.svd(S, compute_uv=False)
    assert np.allclose(sig[: ref.size], ref, rtol=1e-8)


@pytest.mark.parametrize("shape", [(2_000, 37, 5), (70_000, 130, 61), (9, 200_000, 66), (150, 3, 1),
                                   (80, 1_000, 80), (5_000, 33, 75)])
def test_tc_matmul_strided_operands_match_fp64(shape):
    """The reduced-basis stage's DMMA contractions (hc_dgemm): tall x small projections,
    long-inner-dimension products B^T W, transposed / sliced operands in place."""
    import torch
    from paper_1704_04139_b200 import pod
    m, k, n = shape
    g = torch.Generator(device="cuda").manual_seed(9)
    X = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g)
    Y = torch.randn(k, n + 3, dtype=torch.float64, device="cuda", generator=g)[:, 1:n + 1]   # strided slice
    for a, b in ((X, Y), (X.t().contiguous().t(), Y), (Y.t(), X.t()) if m == k else (X, Y)):
        C = pod.tc_matmul(a, b)
        ref = a.cpu().numpy() @ b.cpu().numpy()
        assert np.max(np.abs(C.cpu().numpy() - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1.0) * np.sqrt(k)
    w = torch.rand(k, dtype=torch.float64, device="cuda", generator=g) + 0.5
    Cw = pod.tc_matmul(X, Y, w)
    ref = (X.cpu().numpy() * w.cpu().numpy()) @ Y.cpu().numpy()
    assert np.max(np.abs(Cw.cpu().numpy() - ref)) <= 1e-12 * np.max(np.abs(ref)) * np.sqrt(k)
