"""CPU oracle of the full-order implicit step — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy/scipy, the algorithm of the reference package
``halfcell`` (arXiv 1704.04139 desk-scale implementation, mounted at
/root/reference/pkg) for the hot path this repository accelerates.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it — always as the checker or the
CPU baseline, never as the product path.

Pinned against the reference itself: ``tests/golden/make_golden.py`` runs the
reference in the build container and commits its outputs as fixtures;
``tests/test_oracle_golden.py`` checks this oracle against them.

Reference citations (file:line under pkg/src/halfcell/):
  fvm/dofmap.py:57-101       numbering + validation          -> OracleOperator._number
  fvm/operator.py:121-242    face classification / A_lin     -> OracleOperator._faces
  fvm/operator.py:246-327    interface kinetics + 1/c faces  -> _bv/_ce/_strip/_elel
  fvm/operator.py:331-389    apply and its parts             -> OracleOperator.apply*
  fvm/operator.py:402-471    analytic Jacobian               -> OracleOperator.jacobian
  fvm/newton.py:62-206       Newton, floor, initial potential-> newton_solve / solve_initial_potential
  fvm/timestepping.py:50-106  step + plated update             -> step
  fvm/state.py:44-69, qoi.py  initial fields, QoIs             -> initial_fields / qoi_vectors
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from scipy import ndimage

EL, GR, PL, FOIL, CW, CC = range(6)
NAMES = ("ELECTROLYTE", "GRAPHITE", "PLATED_LI", "LI_FOIL", "COLLECTOR_WORKING",
         "COLLECTOR_COUNTER")
# interface kinds: 0 same phase, 1 BV, 2 counter exchange, 3 stripping, 4 blocking,
# 5 conductor contact, 6 forbidden  (echem/interfaces.py:27-61)
_PAIR_KIND = {
    frozenset((GR, EL)): 1, frozenset((EL, FOIL)): 2, frozenset((EL, PL)): 3,
    frozenset((EL, CW)): 4, frozenset((EL, CC)): 4, frozenset((GR, FOIL)): 6,
    frozenset((PL, FOIL)): 6,
}
KIND = np.full((6, 6), 5, dtype=np.int8)
for _a in range(6):
    KIND[_a, _a] = 0
    for _b in range(6):
        if _a != _b and frozenset((_a, _b)) in _PAIR_KIND:
            KIND[_a, _b] = _PAIR_KIND[frozenset((_a, _b))]


class OracleError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind   # "ModelError", "NumericsError", "NonConvergence", "SimulationError"


class Params:
    """Plain-attribute parameter set (same names as MaterialParams, params.py:50-113)."""

    def __init__(self, src=None, **kw):
        defaults = dict(temperature=298.15, d_gr=5.0e-13, sigma_gr=50.0, sigma_li=2.0e3,
                        sigma_cc=2.0e3, sigma_pl=2.0e3, d_el=3.0e-10, kappa_el=1.0, t_plus=0.26,
                        dlnf_dlnc=0.0, i00_grel=2.0e-4, i00_ceel=50.0, i00_plel=2.0,
                        c_gr_max=30000.0, n_const_thickness=0.48e-9, c_li_metal=76900.0,
                        c_el_init=1000.0, soc_init=0.75, F=96485.33, R=8.3145,
                        ocp_table=((0.00, 0.600), (0.04, 0.400), (0.10, 0.280), (0.20, 0.220),
                                   (0.30, 0.210), (0.45, 0.185), (0.55, 0.155), (0.65, 0.150),
                                   (0.80, 0.145), (0.90, 0.100), (0.97, 0.070), (1.00, 0.060)))
        if src is not None:
            for k in defaults:
                if k in ("F", "R"):
                    defaults[k] = getattr(src.constants, k)
                else:
                    defaults[k] = getattr(src, k)
        defaults.update(kw)
        self.__dict__.update(defaults)
        tab = np.asarray(self.ocp_table, dtype=float)
        self.knots, self.vals = tab[:, 0], tab[:, 1]

    @property
    def vt(self):
        return 2.0 * self.R * self.temperature / self.F

    def ocp(self, c):
        return np.interp(np.asarray(c, float) / self.c_gr_max, self.knots, self.vals)

    def ocp_slope(self, c):
        s = np.asarray(c, float) / self.c_gr_max
        seg = np.clip(np.searchsorted(self.knots, s, side="right") - 1, 0, self.knots.size - 2)
        d = (self.vals[seg + 1] - self.vals[seg]) / (self.knots[seg + 1] - self.knots[seg])
        return np.where((s < self.knots[0]) | (s > self.knots[-1]), 0.0, d / self.c_gr_max)


def f_pre(n, nc):
    n4 = np.asarray(n, float) ** 4
    return n4 / (nc ** 4 + n4)


def f_pre_deriv(n, nc):
    n = np.asarray(n, float)
    return 4.0 * n ** 3 * nc ** 4 / (nc ** 4 + n ** 4) ** 2


class OracleOperator:
    """numpy restatement of SystemOperator on a labels array [z, y, x]."""

    def __init__(self, labels: np.ndarray, voxel_size_um: float, p: Params):
        self.labels = np.ascontiguousarray(labels, dtype=np.uint8)
        self.p = p
        self.h = voxel_size_um * 1e-6
        self.face_area = self.h * self.h
        self.n_const = p.c_li_metal * p.n_const_thickness * self.face_area
        self.sc = 1.0 / (p.F * self.h)
        self._number()
        self._faces()

    # -- numbering and validation (dofmap.py:57-101) ------------------------------
    def _number(self):
        lab = self.labels
        flat = lab.ravel()
        nz = lab.shape[0]
        if not np.any(flat == GR):
            raise OracleError("ModelError", "grid contains no graphite electrode")
        if not np.any(flat == FOIL):
            raise OracleError("ModelError", "grid contains no lithium foil counter electrode")
        six = ndimage.generate_binary_structure(3, 1)
        comp, ncomp = ndimage.label(lab == EL, structure=six)
        ok = False
        if ncomp:
            a = np.unique(comp[ndimage.binary_dilation(lab == GR, six) & (lab == EL)])
            b = np.unique(comp[ndimage.binary_dilation(lab == FOIL, six) & (lab == EL)])
            ok = np.intersect1d(a, b).size > 0
        if not ok:
            raise OracleError("ModelError",
                              "no electrolyte path connects the electrode to the counter electrode")
        grounded = np.zeros(lab.shape, dtype=bool)
        grounded[nz - 1] = lab[nz - 1] == CC
        if not grounded[nz - 1].any():
            raise OracleError("ModelError", "outermost z layer holds no counter collector to ground")
        gflat = grounded.ravel()
        cmask = (flat == GR) | (flat == EL)
        self.c_dof = np.where(cmask, np.cumsum(cmask) - 1, -1).astype(np.int64)
        pmask = ~gflat
        self.p_dof = np.where(pmask, np.cumsum(pmask) - 1, -1).astype(np.int64)
        self.n_c, self.n_p = int(cmask.sum()), int(pmask.sum())
        self.n = self.n_c + self.n_p
        self.plated = np.flatnonzero(flat == PL)
        self.dirichlet = np.flatnonzero(gflat)
        self.slot_of = np.full(flat.size, -1, dtype=np.int64)
        self.slot_of[self.plated] = np.arange(self.plated.size)

    # -- faces (operator.py:121-242) -------------------------------------------------
    def _faces(self):
        lab, p = self.labels, self.p
        nz, ny, nx = lab.shape
        ids = np.arange(lab.size).reshape(lab.shape)
        lo = np.concatenate([ids[:-1].ravel(), ids[:, :-1].ravel(), ids[:, :, :-1].ravel()])
        hi = np.concatenate([ids[1:].ravel(), ids[:, 1:].ravel(), ids[:, :, 1:].ravel()])
        flat = lab.ravel()
        a, b = flat[lo].astype(np.int64), flat[hi].astype(np.int64)
        kind = KIND[a, b]
        g_lo, g_hi = self.p_dof[lo] < 0, self.p_dof[hi] < 0
        bad = (kind == 6) & ~(g_lo & g_hi)
        if bad.any():
            f = np.flatnonzero(bad)[0]
            raise OracleError("ModelError", f"{NAMES[a[f]]} and {NAMES[b[f]]} voxels share a face; "
                              "this adjacency is geometrically forbidden")
        one = g_lo ^ g_hi
        if np.any(one & np.isin(kind, (1, 2, 3))):
            raise OracleError("ModelError", "interface kinetics on a grounded face are not supported")
        sig = np.array([p.kappa_el, p.sigma_gr, p.sigma_pl, p.sigma_li, p.sigma_cc, p.sigma_cc])
        gF2 = 1.0 / (p.F * self.h * self.h)
        xc = self.c_dof
        xp = np.where(self.p_dof >= 0, self.n_c + self.p_dof, -1)
        rows, cols, vals = [], [], []

        def put(r, c, v):
            rows.append(np.asarray(r, np.int64))
            cols.append(np.asarray(c, np.int64))
            vals.append(np.broadcast_to(np.asarray(v, float), np.shape(r)).copy())

        def pair(i, j, g):  # two-point flux g (x_i - x_j) on row i and its mirror on row j
            put(i, i, g); put(i, j, -g); put(j, j, g); put(j, i, -g)

        harm = 2.0 * sig[a] * sig[b] / (sig[a] + sig[b]) * gF2
        sel = one & np.isin(kind, (0, 5))
        live = np.where(g_lo, hi, lo)[sel]
        put(xp[live], xp[live], harm[sel])
        inner = ~g_lo & ~g_hi
        same = inner & (kind == 0)
        for ph in range(6):
            m = same & (a == ph)
            if not m.any():
                continue
            if ph == GR:
                pair(xc[lo[m]], xc[hi[m]], p.d_gr / self.h ** 2)
            if ph == EL:
                pair(xc[lo[m]], xc[hi[m]], p.d_el / self.h ** 2)
                gm = p.t_plus * p.kappa_el * gF2
                ci, cj, pi, pj = xc[lo[m]], xc[hi[m]], xp[lo[m]], xp[hi[m]]
                put(ci, pi, gm); put(ci, pj, -gm); put(cj, pj, gm); put(cj, pi, -gm)
            pair(xp[lo[m]], xp[hi[m]], sig[ph] * gF2)
        m = inner & (kind == 5)
        pair(xp[lo[m]], xp[hi[m]], harm[m])
        r = np.concatenate(rows) if rows else np.empty(0, np.int64)
        c = np.concatenate(cols) if cols else np.empty(0, np.int64)
        v = np.concatenate(vals) if vals else np.empty(0)
        self.A_lin = sp.csr_matrix((v, (r, c)), shape=(self.n, self.n))
        self.A_lin_abs = abs(self.A_lin)

        def oriented(k):
            m = inner & (kind == k)
            el_first = a[m] == EL
            return np.where(el_first, hi[m], lo[m]), np.where(el_first, lo[m], hi[m])

        so, el = oriented(1)
        self.bv = (xc[so], xc[el], xp[so], xp[el])
        so, el = oriented(2)
        self.ce = (xp[so], xc[el], xp[el])
        so, el = oriented(3)
        self.strip = (xp[so], xc[el], xp[el], self.slot_of[so])
        m = same & (a == EL)
        self.elel = (xc[lo[m]], xc[hi[m]], xp[lo[m]], xp[hi[m]])
        self.gX = (p.kappa_el * (p.t_plus - 1.0) * p.R * p.temperature * (1.0 + p.dlnf_dlnc)
                   / (p.F ** 2 * self.h ** 2))
        drive = np.flatnonzero(flat[: nx * ny] == CW)
        self.b_bnd = np.zeros(self.n)
        self.b_bnd[xp[drive]] = -1.0 / (p.F * self.h)
        self.n_drive_faces = int(drive.size)

    # -- interface kinetics (operator.py:246-327) ------------------------------------
    def _bv(self, cg, ce, pg, pe, jac=False):
        p = self.p
        eta = pg - p.ocp(cg) - pe
        rt = np.sqrt(cg * ce)
        s = np.sinh(eta / p.vt)
        i = 2.0 * p.i00_grel * rt * s
        if not jac:
            return i
        ch = np.cosh(eta / p.vt)
        return i, (2.0 * p.i00_grel * (0.5 * np.sqrt(ce / cg) * s - rt * ch * p.ocp_slope(cg) / p.vt),
                   p.i00_grel * np.sqrt(cg / ce) * s, 2.0 * p.i00_grel * rt * ch / p.vt)

    def _ce(self, pf, pe, jac=False):
        p = self.p
        i = 2.0 * p.i00_ceel * np.sinh((pf - pe) / p.vt)
        return (i, 2.0 * p.i00_ceel * np.cosh((pf - pe) / p.vt) / p.vt) if jac else i

    def _strip(self, ce, pp, pe, n, beta=0.0, jac=False):
        p, nc = self.p, self.n_const
        arg = (pp - pe) / p.vt
        ex, emx = np.exp(arg), np.exp(-arg)
        E = p.i00_plel * np.sqrt(ce)
        if beta == 0.0:
            fp = f_pre(n, nc)
            i = E * (fp * ex - emx)
            return (i, (0.5 * i / ce, E * (fp * ex + emx) / p.vt)) if jac else i
        lo, hi = -E * emx, E * (ex - emx)
        i = np.clip(E * (f_pre(n, nc) * ex - emx), lo, hi)
        for _ in range(60):
            ne = np.maximum(n - beta * i, 0.0)
            fd = np.where(ne > 0, f_pre_deriv(ne, nc), 0.0)
            step = (i - E * (f_pre(ne, nc) * ex - emx)) / (1.0 + E * ex * fd * beta)
            i_new = np.clip(i - step, lo, hi)
            done = np.max(np.abs(i_new - i), initial=0.0) <= 1e-14 * (1.0 + np.max(np.abs(i_new), initial=0.0))
            i = i_new
            if done:
                break
        if not jac:
            return i
        ne = np.maximum(n - beta * i, 0.0)
        f = f_pre(ne, nc)
        gi = 1.0 + E * ex * np.where(ne > 0, f_pre_deriv(ne, nc), 0.0) * beta
        return i, ((0.5 / ce) * E * (f * ex - emx) / gi, E * (f * ex + emx) / p.vt / gi)

    # -- evaluations (operator.py:331-389) ----------------------------------------------
    def apply_bv(self, x, n_pl, beta=0.0):
        out = np.zeros(self.n)
        with np.errstate(invalid="ignore"):
            cg, ce, pg, pe = self.bv
            if cg.size:
                q = self.sc * self._bv(x[cg], x[ce], x[pg], x[pe])
                for rr, sgn in ((cg, 1), (pg, 1), (ce, -1), (pe, -1)):
                    np.add.at(out, rr, sgn * q)
            pf, ce, pe = self.ce
            if pf.size:
                q = self.sc * self._ce(x[pf], x[pe])
                for rr, sgn in ((pf, 1), (ce, -1), (pe, -1)):
                    np.add.at(out, rr, sgn * q)
            pp, ce, pe, slot = self.strip
            if pp.size:
                q = self.sc * self._strip(x[ce], x[pp], x[pe], n_pl[slot], beta)
                for rr, sgn in ((pp, 1), (ce, -1), (pe, -1)):
                    np.add.at(out, rr, sgn * q)
        return out

    def apply_one_over_c(self, x):
        out = np.zeros(self.n)
        ci, cj, pi, pj = self.elel
        if ci.size:
            with np.errstate(invalid="ignore", divide="ignore"):
                q = self.gX * (np.log(x[cj]) - np.log(x[ci]))
            tp = self.p.t_plus
            np.add.at(out, pi, -q)
            np.add.at(out, pj, q)
            np.add.at(out, ci, -tp * q)
            np.add.at(out, cj, tp * q)
        return out

    def apply_lin(self, x):
        return self.A_lin @ x

    def apply(self, x, n_pl, mu, beta=0.0):
        out = mu * self.b_bnd + self.A_lin @ x + self.apply_bv(x, n_pl, beta) + self.apply_one_over_c(x)
        if not np.all(np.isfinite(out)):
            raise OracleError("NumericsError", "operator produced a non-finite value")
        return out

    def row_scale(self, x, n_pl, mu, beta=0.0):
        """Sum of |contributions| per row: the yardstick of floating-point agreement."""
        s = self.A_lin_abs @ np.abs(x) + np.abs(mu * self.b_bnd)
        cg, ce, pg, pe = self.bv
        if cg.size:
            q = np.abs(self.sc * self._bv(x[cg], x[ce], x[pg], x[pe]))
            for rr in (cg, pg, ce, pe):
                np.add.at(s, rr, q)
        pf, ce, pe = self.ce
        if pf.size:
            q = np.abs(self.sc * self._ce(x[pf], x[pe]))
            for rr in (pf, ce, pe):
                np.add.at(s, rr, q)
        pp, ce, pe, slot = self.strip
        if pp.size:
            q = np.abs(self.sc * self._strip(x[ce], x[pp], x[pe], n_pl[slot], beta))
            for rr in (pp, ce, pe):
                np.add.at(s, rr, q)
        ci, cj, pi, pj = self.elel
        if ci.size:
            q = np.abs(self.gX * (np.log(x[cj]) - np.log(x[ci])))
            for rr in (ci, cj, pi, pj):
                np.add.at(s, rr, q)
        return s

    # -- Jacobian (operator.py:402-471) ----------------------------------------------------
    def jacobian(self, x, n_pl, beta=0.0):
        R, C, V = [], [], []

        def ent(rows, col, v):
            R.append(rows); C.append(col); V.append(np.broadcast_to(v, rows.shape))

        sc = self.sc
        cg, ce, pg, pe = self.bv
        if cg.size:
            _, (a, b, g) = self._bv(x[cg], x[ce], x[pg], x[pe], jac=True)
            for rr, s in ((cg, 1.0), (pg, 1.0), (ce, -1.0), (pe, -1.0)):
                ent(rr, cg, s * sc * a); ent(rr, ce, s * sc * b)
                ent(rr, pg, s * sc * g); ent(rr, pe, -s * sc * g)
        pf, cel, pel = self.ce
        if pf.size:
            _, g = self._ce(x[pf], x[pel], jac=True)
            for rr, s in ((pf, 1.0), (cel, -1.0), (pel, -1.0)):
                ent(rr, pf, s * sc * g); ent(rr, pel, -s * sc * g)
        pp, cel, pel, slot = self.strip
        if pp.size:
            _, (b, g) = self._strip(x[cel], x[pp], x[pel], n_pl[slot], beta, jac=True)
            for rr, s in ((pp, 1.0), (cel, -1.0), (pel, -1.0)):
                ent(rr, cel, s * sc * b); ent(rr, pp, s * sc * g); ent(rr, pel, -s * sc * g)
        ci, cj, pi, pj = self.elel
        if ci.size:
            di, dj = -self.gX / x[ci], self.gX / x[cj]
            tp = self.p.t_plus
            for rr, s in ((pi, -1.0), (pj, 1.0), (ci, -tp), (cj, tp)):
                ent(rr, ci, s * di); ent(rr, cj, s * dj)
        if not R:
            return self.A_lin.copy()
        J = sp.csr_matrix((np.concatenate(V), (np.concatenate(R), np.concatenate(C))),
                          shape=(self.n, self.n))
        return (self.A_lin + J).tocsr()

    # -- plated fluxes (timestepping.py:50-57) -------------------------------------------
    def plated_flux(self, x, n_pl, beta):
        flux = np.zeros(n_pl.size)
        pp, ce, pe, slot = self.strip
        if pp.size:
            i = self._strip(x[ce], x[pp], x[pe], n_pl[slot], beta)
            np.add.at(flux, slot, i * self.face_area / self.p.F)
        return flux


# ---- initial fields and QoIs (state.py:44-69, qoi.py:11-34) ---------------------------
def initial_fields(op: OracleOperator):
    p, flat = op.p, op.labels.ravel()
    x = np.zeros(op.n)
    cv = np.flatnonzero(op.c_dof >= 0)
    x[op.c_dof[cv]] = np.where(flat[cv] == GR, p.soc_init * p.c_gr_max, p.c_el_init)
    pv = np.flatnonzero(op.p_dof >= 0)
    work = np.isin(flat[pv], (GR, PL, CW))
    x[op.n_c + op.p_dof[pv[work]]] = p.ocp(p.soc_init * p.c_gr_max)
    n_pl = np.full(op.plated.size, op.h ** 3 * p.c_li_metal)
    return x, n_pl


def qoi_vectors(op: OracleOperator):
    flat = op.labels.ravel()
    nxy = op.labels.shape[1] * op.labels.shape[2]
    v_cp = np.zeros(op.n)
    outer = np.flatnonzero(flat[:nxy] == CW)
    if outer.size:
        v_cp[op.n_c + op.p_dof[outer]] = 1.0 / outer.size
    v_ac = np.zeros(op.n)
    gr = np.flatnonzero(flat == GR)
    v_ac[op.c_dof[gr]] = 1.0 / gr.size
    return v_cp, v_ac


# ---- Newton (newton.py:62-206) -------------------------------------------------------
def _floor(op, x, inv_dt=0.0):
    s = op.A_lin_abs @ np.abs(x)
    if inv_dt:
        s[: op.n_c] += np.abs(x[: op.n_c]) * inv_dt
    return 1e-13 * float(np.linalg.norm(s))


def _solve(J, rhs):
    return spla.splu(J.tocsc()).solve(rhs)


def newton_solve(op, x_guess, dt, x_prev, n_pl, mu, rtol=1e-9, atol=1e-10, max_iter=20,
                 implicit_plated=True):
    nc, inv_dt = op.n_c, 1.0 / dt
    beta = dt * op.face_area / op.p.F if implicit_plated else 0.0
    mass = sp.diags(np.r_[np.full(nc, inv_dt), np.zeros(op.n_p)])

    def res(x):
        r = op.apply(x, n_pl, mu, beta)
        r[:nc] += (x[:nc] - x_prev[:nc]) * inv_dt
        return r

    x = x_guess.copy()
    try:
        r = res(x)
    except OracleError as e:
        raise OracleError("NonConvergence", f"initial residual not evaluable: {e}")
    norm = norm0 = float(np.linalg.norm(r))
    tol = max(atol, rtol * norm0, _floor(op, x, inv_dt))
    norms, it = [norm0], 0
    if norm0 <= tol:
        return x, 0, norms
    for it in range(1, max_iter + 1):
        d = _solve(op.jacobian(x, n_pl, beta) + mass, -r)
        alpha = 1.0
        neg = d[:nc] < 0
        if neg.any():
            alpha = min(alpha, 0.99 * np.min(x[:nc][neg] / -d[:nc][neg]))
        if alpha <= 0:
            raise OracleError("NonConvergence", "positivity guard blocked the Newton step")
        for _ in range(9):
            xt = x + alpha * d
            try:
                rt = res(xt)
                nt = float(np.linalg.norm(rt))
            except OracleError:
                nt = np.inf
            if np.isfinite(nt) and (nt <= norm or nt <= tol):
                break
            alpha *= 0.5
        else:
            xt = x + alpha * d
            rt = res(xt)
            nt = float(np.linalg.norm(rt))
        x, r, norm = xt, rt, nt
        norms.append(norm)
        if norm <= tol:
            return x, it, norms
    raise OracleError("NonConvergence", f"Newton did not reach tolerance {tol:.3e}")


def solve_initial_potential(op, x0, n_pl, mu, rtol=1e-9, atol=1e-10, max_iter=20):
    nc = op.n_c
    x = x0.copy()
    r = op.apply(x, n_pl, mu)[nc:]
    norm = norm0 = float(np.linalg.norm(r))
    tol = max(atol, rtol * norm0, _floor(op, x))
    if norm0 <= tol:
        return x
    for _ in range(max_iter):
        J = op.jacobian(x, n_pl)[nc:, nc:]
        d = _solve(J, -r)
        alpha = 1.0
        for _ in range(9):
            xt = x.copy()
            xt[nc:] += alpha * d
            try:
                rt = op.apply(xt, n_pl, mu)[nc:]
                nt = float(np.linalg.norm(rt))
            except OracleError:
                nt = np.inf
            if np.isfinite(nt) and (nt <= norm or nt <= tol):
                break
            alpha *= 0.5
        x, r, norm = xt, rt, nt
        if norm <= tol:
            return x
    raise OracleError("NonConvergence", f"stationary potential solve stalled at residual {norm:.3e}")


def step(op, x, n_pl, dt, mu, implicit_plated=True, **kw):
    """One fixed-size implicit-Euler step + explicit plated update (timestepping.py:64-106)."""
    xn, it, _ = newton_solve(op, x, dt, x, n_pl, mu, implicit_plated=implicit_plated, **kw)
    beta = dt * op.face_area / op.p.F if implicit_plated else 0.0
    if n_pl.size:
        n_new = n_pl - dt * op.plated_flux(xn, n_pl, beta)
        clamped = float(-n_new[n_new < 0].sum())
        n_new = np.maximum(n_new, 0.0)
    else:
        n_new, clamped = n_pl.copy(), 0.0
    return xn, n_new, it, clamped
