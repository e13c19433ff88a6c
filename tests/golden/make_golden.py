"""Generate golden fixtures by running the REFERENCE implementation (build container only).

    python tests/golden/make_golden.py            # needs /root/reference/pkg/src

Each fixture ``<case>.npz`` holds the reference's own outputs on a small grid:
labels, Dofmap arrays, face lists, operator parts at a perturbed state, a
Jacobian-vector product, the Jacobian sparsity pattern and a short transient
(cell voltage, mean solid concentration, plated inventory per step).  The
files are committed; the GPU box never reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from halfcell.echem import MaterialParams as RefParams  # noqa: E402
from halfcell.fvm import (SolverConfig, SystemOperator, build_dofmap, newton_solve,  # noqa: E402
                          prepare_initial_state, qoi_cell_voltage, qoi_mean_solid_conc, step)
from halfcell.fvm.state import initial_fields  # noqa: E402
from halfcell.microgen import GenConfig, PhaseGrid, generate  # noqa: E402

from paper_1704_04139_b200.microgen import CellSpec, generate_cell  # noqa: E402


def cases():
    g1 = generate(GenConfig(domain_size=(15.0, 15.0, 30.0), voxel_size=1.5, rng_seed=7,
                            plating_intensity=0.05))
    yield "refgen_10x10x20", g1.labels, g1.voxel_size, RefParams(), -20.0, 1.0
    spec = CellSpec(16, 16, 24, 12, 4, seed=3, radius_mean=3.0, porosity=0.35,
                    plating_intensity=0.05)
    g2 = generate_cell(spec)
    p2 = RefParams(soc_init=0.1, i00_plel=1e-3 / np.sqrt(1000.0))
    yield "balls_16x16x24", g2.labels, g2.voxel_size, p2, -8.0, 0.5


def main():
    for name, labels, h, params, mu, dt in cases():
        grid = PhaseGrid(labels, h)
        dof = build_dofmap(grid)
        op = SystemOperator(dof, params)
        rng = np.random.default_rng(11)
        st0 = initial_fields(dof, params)
        x = st0.x.copy()
        x[: dof.n_c] *= 1.0 + 0.05 * rng.standard_normal(dof.n_c)
        x[dof.n_c:] += 0.01 * rng.standard_normal(dof.n_p)
        n_pl = st0.n_pl * rng.uniform(0.0, 1.5, st0.n_pl.size)
        if n_pl.size:
            n_pl[0] = 0.0
        beta = dt * op.face_area / params.constants.F
        v = rng.standard_normal(dof.n_total)
        J = op.jacobian(x, n_pl, mu, beta=beta).tocsr()
        J.sort_indices()
        out = dict(
            labels=labels, voxel_size=h, mu=mu, dt=dt, beta=beta,
            params=np.array([params.soc_init, params.i00_plel]),
            c_dof=dof.c_dof, p_dof=dof.p_dof, plated=dof.plated_voxels, dirichlet=dof.dirichlet,
            bv=np.stack([op.bv_xc_gr, op.bv_xc_el, op.bv_xp_gr, op.bv_xp_el]),
            ce=np.stack([op.ce_xp_fo, op.ce_xc_el, op.ce_xp_el]),
            strip=np.stack([op.strip_xp_pl, op.strip_xc_el, op.strip_xp_el, op.strip_slot]),
            elel=np.stack([op.elel_xc_i, op.elel_xc_j, op.elel_xp_i, op.elel_xp_j]),
            x=x, n_pl=n_pl, v=v,
            apply=op.apply(x, n_pl, mu, beta=beta), apply_bv=op.apply_bv(x, n_pl, beta=beta),
            apply_1c=op.apply_one_over_c(x), apply_lin=op.apply_lin(x), b_bnd=op.b_bnd,
            jv=J @ v, j_indptr=J.indptr, j_indices=J.indices,
        )
        # one Newton solve from the perturbed state
        cfg = SolverConfig()
        res = newton_solve(op, x, dt, x, n_pl, mu, cfg)
        out["newton_x"] = res.x
        out["newton_iters"] = res.n_iter
        # short transient with fixed steps from the stationary initial state
        state = prepare_initial_state(op, params, mu, cfg)
        traj_v, traj_c, traj_n, xs = [], [], [], [state.x]
        traj_v.append(qoi_cell_voltage(state, dof))
        traj_c.append(qoi_mean_solid_conc(state, dof))
        traj_n.append(state.n_pl.sum())
        for _ in range(4):
            state, dt_used, _, info = step(op, state, dt, mu, cfg)
            assert abs(dt_used - dt) < 1e-15 and info.retries == 0
            traj_v.append(qoi_cell_voltage(state, dof))
            traj_c.append(qoi_mean_solid_conc(state, dof))
            traj_n.append(state.n_pl.sum())
            xs.append(state.x)
        out.update(traj_voltage=np.array(traj_v), traj_mean_c=np.array(traj_c),
                   traj_npl=np.array(traj_n), traj_x0=xs[0], traj_xend=xs[-1],
                   traj_npl_end=state.n_pl)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(name, labels.shape, dof.describe(), "bv", op.bv_xc_gr.size, "strip",
              op.strip_slot.size, "->", os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
