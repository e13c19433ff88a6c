"""CPU oracle of the reduced-order online stage — TEST INFRASTRUCTURE ONLY.

numpy/scipy restatement of ``hc_rom_run`` (paper_1704_04139_b200/csrc/hc_rom.cu):
the reduced implicit-Euler / chord-Newton loop of SPEC ``mor.solve_rom`` (arXiv
1704.04139 Eq. 20) on the data of a ``ReducedModel`` (``ReducedModel.host()``).  The
face kinetics are the reference's (operator.py:246-327), taken from
``oracle.fvm_oracle.OracleOperator`` so the reduced model is checked against the
same restatement the full-order path is pinned to.  The reference tree has no
``mor`` package, so this stage is "parity unpinned" against reference code: it is
pinned by construction tests instead (identity-like bases reproduce the full-order
trajectory, EI exactness at the interpolation rows, see tests/test_gpu_rom.py).

Also holds ``deim`` (sequential DEIM greedy, the definition the GPU blocked version
must reproduce).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla

RF_BV, RF_CE, RF_STRIP, RF_ELEL = 0, 1, 2, 3


def deim(W: np.ndarray) -> np.ndarray:
    """Sequential DEIM: for column l, the row of max |W_l - I_{l-1}[W_l]| (first on ties)."""
    n, m = W.shape
    pi = []
    for l in range(m):
        r = W[:, l].copy()
        if l:
            P = np.asarray(pi)
            r -= W[:, :l] @ np.linalg.solve(W[P, :l], W[P, l])
        pi.append(int(np.argmax(np.abs(r))))
    return np.asarray(pi, dtype=np.int64)


def _faces(op, d, xs, npl, beta, need_d):
    """q_f and dq_f/d(stencil dofs) for every active face (hc_rom.cu rom_face)."""
    kind, fd, slot = d["f_kind"], d["f_dof"].reshape(-1, 4), d["f_slot"]
    n_f = kind.size
    q = np.zeros(n_f)
    dq = np.zeros((n_f, 4))
    sc = op.sc
    for kd in (RF_BV, RF_CE, RF_STRIP, RF_ELEL):
        f = np.flatnonzero(kind == kd)
        if not f.size:
            continue
        a = fd[f]
        if kd == RF_BV:
            i, (da, db, dg) = op._bv(xs[a[:, 0]], xs[a[:, 1]], xs[a[:, 2]], xs[a[:, 3]], jac=True)
            q[f] = sc * i
            dq[f, 0], dq[f, 1], dq[f, 2], dq[f, 3] = sc * da, sc * db, sc * dg, -sc * dg
        elif kd == RF_CE:
            i, dg = op._ce(xs[a[:, 0]], xs[a[:, 2]], jac=True)
            q[f] = sc * i
            dq[f, 0], dq[f, 2] = sc * dg, -sc * dg
        elif kd == RF_STRIP:
            i, (dce, dpp) = op._strip(xs[a[:, 1]], xs[a[:, 0]], xs[a[:, 2]], npl[slot[f]], beta, jac=True)
            q[f] = sc * i
            dq[f, 0], dq[f, 1], dq[f, 2] = sc * dpp, sc * dce, -sc * dpp
        else:
            ci, cj = xs[a[:, 0]], xs[a[:, 1]]
            q[f] = op.gX * (np.log(cj) - np.log(ci))
            dq[f, 0], dq[f, 1] = -op.gX / ci, op.gX / cj
    return q, dq


def rom_run(op, d: dict, xt, npl, mu, dt, n_steps, rtol=1e-10, max_iter=40, refresh=6, jac_steps=8):
    """Same loop as k_rom_run; returns (xt, n_pl, qoi (n_steps, 2), iters)."""
    k, k_c, m = d["k"], d["k_c"], d["m"]
    A, Mr, bnd, E = (d[n].reshape(k, -1) if n != "bnd" else d[n] for n in ("A", "Mr", "bnd", "E"))
    BS = d["BS"].reshape(-1, k)
    row_ptr, row_face, row_coef = d["row_ptr"], d["row_face"], d["row_coef"]
    fd = d["f_dof"].reshape(-1, 4)
    rows = np.repeat(np.arange(m), np.diff(row_ptr))
    xt = np.array(xt, dtype=float)
    npl = np.array(npl, dtype=float)
    inv_dt = 1.0 / dt
    beta = dt * op.face_area / op.p.F
    qoi = np.zeros((n_steps, 2))
    iters = np.zeros(n_steps, np.int64)
    lu = None
    since, prev_it = 0, 0
    for step in range(n_steps):
        xo = xt.copy()
        conv = False
        it = 0
        step_fresh = step == 0 or since >= jac_steps or prev_it > refresh
        while it < max_iter and not conv:
            fresh = (it == 0 and step_fresh) or (refresh > 0 and it > 0 and it % refresh == 0)
            if fresh:
                since = 0
            xs = BS @ xt
            q, dq = _faces(op, d, xs, npl, beta, fresh)
            N = np.zeros(m)
            np.add.at(N, rows, row_coef * q[row_face])
            r = Mr @ (xt - xo) * inv_dt + A @ xt + mu * bnd + E @ N
            if fresh:
                G = np.zeros((m, k))
                for c in range(4):
                    dd = fd[row_face, c]
                    ok = dd >= 0
                    np.add.at(G, rows[ok], (row_coef[ok] * dq[row_face[ok], c])[:, None] * BS[dd[ok]])
                lu = sla.lu_factor(A + Mr * inv_dt + E @ G)
            delta = sla.lu_solve(lu, r)
            xn = xt - delta
            dc, dp = np.linalg.norm(delta[:k_c]), np.linalg.norm(delta[k_c:])
            conv = dc <= rtol * np.linalg.norm(xn[:k_c]) and dp <= rtol * (np.linalg.norm(xn[k_c:]) + 1.0)
            if not (np.isfinite(dc) and np.isfinite(dp)):
                raise FloatingPointError(f"non-finite reduced update at step {step}")
            xt = xn
            it += 1
        if not conv:
            raise RuntimeError(f"reduced Newton did not converge at step {step}")
        since += 1
        prev_it = it
        xs = BS @ xt
        q, _ = _faces(op, d, xs, npl, beta, False)
        flux = np.zeros(npl.size)
        for s in range(d["n_pl"]):
            for e in range(d["pl_ptr"][s], d["pl_ptr"][s + 1]):
                flux[s] += q[d["pl_face"][e]] / op.sc * op.face_area / op.p.F
        npl = np.maximum(npl - dt * flux, 0.0)
        qoi[step] = (d["q_v"] @ xt, d["q_ac"] @ xt)
        iters[step] = it
    return xt, npl, qoi, iters
