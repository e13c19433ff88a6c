"""Generate golden fixtures by running the REFERENCE implementation (build container only).

    python tests/golden/make_golden.py            # needs /root/reference/pkg/src

Each fixture ``<case>.npz`` holds the reference's own outputs on a small grid:
labels, Dofmap arrays, face lists, operator parts at a perturbed state, a
Jacobian-vector product, the Jacobian sparsity pattern, ``A_lin`` (operator.py:221),
the stripping face currents (operator.py:391-399), restricted sub-operator rows and
their local Jacobians (operator.py:476-646), one Newton solve with its iterates and
residual norms and one with a source term (newton.py:86-168), and a short transient
(cell voltage, mean solid concentration, plated inventory per step).  The files are
committed; the GPU box never reads /root/reference.  ``balls_16x16x24`` is built by
this package's ``generate_cell`` (the spec is stored; tests/test_microgen.py checks the
generator still reproduces the labels bit for bit).
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


def plating_cases():
    """Reference germ-grain plating (microgen/plating.py:53-109) on ball-union anodes."""
    import dataclasses
    from halfcell.microgen.plating import plate_germs as ref_plate
    out = {}
    for k, (seed, intensity, radius, h) in enumerate([(5, 0.05, 2.2, 1.0), (6, 0.02, 3.0, 1.0),
                                                       (7, 0.08, 1.5, 0.75)]):
        spec = CellSpec(24, 20, 32, 16, 6, seed=seed, radius_mean=3.0, porosity=0.4,
                        plating_intensity=0.0, voxel_size=h)
        base = generate_cell(dataclasses.replace(spec))
        plated = ref_plate(PhaseGrid(base.labels, h), intensity, radius, np.random.default_rng(100 + k))
        out[f"in_{k}"] = base.labels
        out[f"out_{k}"] = plated.labels
        out[f"args_{k}"] = np.array([intensity, radius, h, 100 + k])
    path = os.path.join(HERE, "plating_ref.npz")
    np.savez_compressed(path, **out)
    print("plating_ref ->", os.path.getsize(path), "bytes")


def main():
    plating_cases()
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
        A = op.A_lin.tocsr()
        A.sort_indices()
        cur, slot = op.strip_face_currents(x, n_pl, beta=beta)
        out = dict(
            a_indptr=A.indptr, a_indices=A.indices, a_data=A.data, strip_current=cur, strip_slot=slot,
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
        out["newton_iterates"] = np.stack(res.iterates)
        out["newton_norms"] = np.array(res.residual_norms)
        # a solve with a source term (newton.py:107-108)
        # a gentle volumetric source on the concentration rows (1e-3 relative per step)
        src = np.zeros(dof.n_total)
        src[: dof.n_c] = 1e-3 * x[: dof.n_c] / dt * rng.standard_normal(dof.n_c)
        res_s = newton_solve(op, x, dt, x, n_pl, mu, cfg, source=src)
        out.update(source=src, source_x=res_s.x, source_iters=res_s.n_iter)
        # restricted sub-operators (the empirical-interpolation access path)
        for which in ("bv", "one_over_c"):
            view = op.sub_operator(which)
            cand = view.output_dofs()
            rows = np.sort(rng.choice(cand, size=min(40, cand.size), replace=False))
            rs = view.restricted(rows)
            xs = x[rs.stencil]
            out[f"sub_{which}_rows"] = rs.rows
            out[f"sub_{which}_stencil"] = rs.stencil
            out[f"sub_{which}_apply"] = rs.apply(xs, n_pl, beta=beta)
            out[f"sub_{which}_jac"] = rs.jacobian(xs, n_pl, beta=beta).toarray()
            out[f"sub_{which}_output_dofs"] = cand
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
