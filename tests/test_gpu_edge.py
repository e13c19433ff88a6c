"""GPU edge cases vs the CPU oracle: 1-D column cells, no plated lithium, plated
lithium everywhere on the surface, ragged (non-multiple-of-tile) grid sizes on both
stencil paths (cp.async for nx % 4 != 0, tensor-map tiles otherwise)."""

import numpy as np
import pytest

from conftest import scaled_err
from oracle import fvm_oracle as O

pytestmark = pytest.mark.gpu

EL, GR, PL, FOIL, CW, CC = range(6)


def column(nz=12):
    lab = np.zeros((nz, 1, 1), dtype=np.uint8)
    lab[0] = CW
    lab[1:4] = GR
    lab[nz - 4:nz - 1] = FOIL
    lab[nz - 1] = CC
    return lab


def slab(nx, ny, nz, plated=True, seed=0):
    rng = np.random.default_rng(seed)
    lab = np.zeros((nz, ny, nx), dtype=np.uint8)
    lab[0] = CW
    e1 = nz // 2
    solid = rng.random((e1 - 2, ny, nx)) < 0.55
    lab[1:e1 - 1][solid] = GR
    lab[1] = GR                       # keep the graphite network on the collector
    if plated:
        top = lab[e1 - 2] == GR
        lab[e1 - 1][top] = PL         # a plated film on the top graphite layer
    lab[nz - 3:nz - 1] = FOIL
    lab[nz - 1] = CC
    return lab


CASES = {
    "column_1x1x12": column(),
    "ragged_7x5x14_no_plating": slab(7, 5, 14, plated=False, seed=1),
    "ragged_33x9x17_plated": slab(33, 9, 17, plated=True, seed=2),
    # tensor-map (TMA) stencil path, nx % 4 == 0, on grids that are not multiples of the
    # 32 x 8 tile: the narrowest grid the path takes, partial tiles in x and y with zero-filled
    # halos, and fewer planes than one CTA's ring of staged planes
    "tma_4x4x10_plated": slab(4, 4, 10, plated=True, seed=4),
    "tma_36x12x9_plated": slab(36, 12, 9, plated=True, seed=5),
    "tma_40x3x21_no_plating": slab(40, 3, 21, plated=False, seed=6),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_edge_geometry_parity(name):
    import paper_1704_04139_b200 as P
    lab = CASES[name]
    params = P.MaterialParams(soc_init=0.4)
    op = P.SystemOperator(P.build_dofmap(P.PhaseGrid(lab, 1.0)), params)
    orc = O.OracleOperator(lab, 1.0, O.Params(soc_init=0.4))
    assert np.array_equal(op.dof.c_dof, orc.c_dof) and np.array_equal(op.dof.p_dof, orc.p_dof)
    rng = np.random.default_rng(3)
    x, n_pl = O.initial_fields(orc)
    x[: orc.n_c] *= 1.0 + 0.05 * rng.standard_normal(orc.n_c)
    x[orc.n_c:] += 0.01 * rng.standard_normal(orc.n_p)
    if n_pl.size:
        n_pl = n_pl * rng.uniform(0.0, 1.5, n_pl.size)
    beta = orc.face_area / orc.p.F
    mu = -3.0
    r = op.apply(x, n_pl, mu, beta=beta)
    assert scaled_err(r, orc.apply(x, n_pl, mu, beta), orc.row_scale(x, n_pl, mu, beta)) < 1e-10
    v = rng.standard_normal(orc.n)
    J = orc.jacobian(x, n_pl, beta)
    assert scaled_err(op.jvp(x, n_pl, v, beta=beta), J @ v, abs(J) @ np.abs(v)) < 1e-10
    # one full Newton solve vs the oracle's SuperLU Newton
    res = P.newton_solve(op, x, 1.0, x, n_pl, mu, P.SolverConfig())
    xo, _, _ = O.newton_solve(orc, x, 1.0, x, n_pl, mu)
    nc = orc.n_c
    assert np.max(np.abs(res.x[:nc] - xo[:nc]) / np.abs(xo[:nc])) < 1e-8
    # the floating working-electrode potential is only determined to Newton tolerance
    # (a near-null mode of the phi block); the curve bar is 1e-6 relative
    assert np.max(np.abs(res.x[nc:] - xo[nc:])) < 1e-6 * max(1.0, np.max(np.abs(xo[nc:])))
