"""Reduced-order model: offline build and online solve (SPEC ``mor``; arXiv 1704.04139 §2.5).

The reference tree does not ship its ``mor`` package; this module follows SPEC
``mor.pod / ei_greedy / build_rom / solve_rom`` and BASELINE config 4:

* snapshots: accepted full-order states of one trajectory (``hc_step``) and the
  nonlinear sub-operator evaluations ``N(x) = A_bv(x) + A_1/c(x)`` at them;
* POD per field (method of snapshots): the Gram matrix on the FP64 tensor cores
  (``hc_pod_gram``), eigendecomposition of the small Gram, basis projection
  ``S U / sigma`` and a CholeskyQR2 re-orthonormalisation ``V R^-1`` — every dense
  contraction of the stage (also the DEIM block updates and ``B^T W``) is a DMMA
  contraction (``hc_dgemm`` through :func:`pod.tc_matmul`);
* empirical interpolation of ``N``: collateral basis = POD of the ``N`` snapshots,
  interpolation DOFs by the DEIM greedy (blocked: one GEMM per block brings the
  block up to date, then rank-1 updates inside it — exactly the sequential greedy);
* projection of the affine blocks (``B^T A_lin B``, mass, boundary), the EI
  projection ``E = B^T W (W_pi)^-1``, the restricted stencil (the faces touching the
  EI rows plus every stripping face, whose plated inventory is carried exactly);
* online: ``hc_rom_run`` — the whole reduced implicit-Euler/Newton time loop in one
  kernel launch (``csrc/hc_rom.cu``); nothing of full-order length is touched.

Design decisions (SPEC ledger): separate c / phi bases (block-diagonal lifting);
one EI space for the sum of the nonlinear sub-operators; DEIM point selection on
the POD basis of the nonlinear snapshots (the greedy over a compressed training
set); chord Newton with the projected analytic Jacobian refreshed every step.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _native
from .errors import ReductionError
from .pod import pod_gram, tc_matmul
from .qoi import qoi_vectors

RF_BV, RF_CE, RF_STRIP, RF_ELEL = 0, 1, 2, 3


# ------------------------------------------------------------------ snapshots
@dataclass
class Snapshots:
    X: object                  # (n_dof, n_s) device states
    N: object                  # (n_dof, n_s) device nonlinear evaluations N = N_bv + N_1c
    n_pl: list = field(default_factory=list)
    beta: float = 0.0
    Nb: object = None          # (n_dof, n_s) A_bv part (separate EI spaces, SPEC build_rom)
    Nc: object = None          # (n_dof, n_s) A_1/c part


def nonlinear_part(op, x, n_pl, beta: float):
    """N(x) = A_bv(x) + A_1/c(x): the sub-operators interpolated by EI (Eq. 18)."""
    return op.apply_bv(x, n_pl, beta=beta) + op.apply_one_over_c(x)


def collect_snapshots(op, x0, n_pl0, mu: float, dt: float, n_steps: int, cfg=None) -> Snapshots:
    """Run ``n_steps`` fixed full-order steps from (x0, n_pl0) and keep every state."""
    from .newton import SolverConfig
    t = _dev.torch()
    # exact-solve Newton by default: inexact linear solves leave ~1e-8 relative noise in
    # the states, which the trailing POD modes then fit (and the reduced Newton amplifies)
    cfg = cfg or SolverConfig(dt_init=dt, dt_max=dt, linear_safety=0.0)
    c = cfg.to_c()
    st = _native.HcNewtonStats()
    x = _dev.to_dev(x0).clone()
    npl = _dev.to_dev(n_pl0 if _dev.numel(n_pl0) else np.zeros(1)).clone()
    beta = dt * op.face_area / op.p.constants.F
    n = op.dof.n_total
    X = t.empty((n, n_steps + 1), dtype=t.float64, device="cuda")
    Nb = t.empty_like(X)
    Nc = t.empty_like(X)
    pls = []
    for s in range(n_steps + 1):
        if s:
            _native.check(_native.lib().hc_step(op.native.handle, _dev.ptr(x), _dev.ptr(npl), 0.0, dt,
                                                float(mu), ctypes.byref(c), ctypes.byref(st),
                                                _dev.stream()))
        X[:, s] = x
        Nb[:, s] = op.apply_bv(x, npl, beta=beta)
        Nc[:, s] = op.apply_one_over_c(x)
        pls.append(npl.clone())
    return Snapshots(X, Nb + Nc, pls, beta, Nb, Nc)


# ------------------------------------------------------------------ POD / DEIM
def _orthonormalize(V):
    """CholeskyQR2 with the tensor-core Gram: V (n, k) -> orthonormal columns, same span."""
    t = _dev.torch()
    for _ in range(2):
        G = _dev.to_dev(pod_gram(V))
        G = 0.5 * (G + G.t())
        R = t.linalg.cholesky(G, upper=True)
        Rinv = t.linalg.solve_triangular(R, t.eye(R.shape[0], dtype=R.dtype, device=R.device), upper=True)
        V = tc_matmul(V, Rinv)                                           # V R^-1 (DMMA)
    return V


def pod_rank(S, k: int | None = None, rel_tol: float | None = None):
    """Orthonormal POD basis of the columns of S (n, n_s), method of snapshots; returns
    (V (n, k'), singular values).  The rank is at most ``k`` and, with ``rel_tol``, the
    smallest one whose discarded energy sum_{i>k} s_i^2 / sum s_i^2 <= rel_tol^2 (SPEC
    mor.pod; the paper uses 1e-7)."""
    t = _dev.torch()
    S = _dev.to_dev(S)
    if not float(t.linalg.vector_norm(S)) > 0.0:
        raise ReductionError("all-zero snapshot set")
    G = _dev.to_dev(pod_gram(S))
    G = 0.5 * (G + G.t())
    lam, U = t.linalg.eigh(G)
    lam, U = lam.flip(0), U.flip(1)
    lam = t.clamp(lam, min=0.0)
    keep = int((lam > lam[0] * 1e-24).sum())
    if rel_tol is not None:
        if not 0.0 < rel_tol < 1.0:
            raise ReductionError("rel_tol must lie in (0, 1)")
        tail = t.flip(t.cumsum(t.flip(lam, [0]), 0), [0])       # tail[j] = sum_{i >= j} lam_i
        ok = (tail <= rel_tol ** 2 * tail[0]).nonzero()
        keep = min(keep, int(ok[0]) if ok.numel() else keep)
    k = max(1, min(int(k) if k is not None else keep, keep))
    sig = t.sqrt(lam)
    V = tc_matmul(S, U[:, :k] / sig[:k])                                  # DMMA
    return _orthonormalize(V), sig


def deim(W, block: int = 16) -> np.ndarray:
    """DEIM interpolation DOFs of the basis W (n, m): for column l the DOF of the largest
    |residual| of W_l interpolated at the points chosen so far (first index on ties)."""
    t = _dev.torch()
    W = _dev.to_dev(W)
    n, m = W.shape
    pi: list[int] = []
    for l0 in range(0, m, block):
        l1 = min(m, l0 + block)
        R = W[:, l0:l1].clone()
        if l0:
            P = t.as_tensor(pi, device="cuda")
            R -= tc_matmul(W[:, :l0], t.linalg.solve(W[P, :l0], W[P, l0:l1]))
        for j in range(l1 - l0):
            r = R[:, j]
            p = int(t.argmax(t.abs(r)))
            if not float(abs(r[p])) > 0.0:
                raise ReductionError(f"EI greedy stagnated at row {l0 + j}")
            pi.append(p)
            if j + 1 < l1 - l0:
                R[:, j + 1:] -= t.outer(r / r[p], R[p, j + 1:])
    return np.asarray(pi, dtype=np.int64)


# ------------------------------------------------------------------ reduced model
@dataclass
class ReducedModel:
    k_c: int
    k_p: int
    m: int
    Vc: object                 # (n_c, k_c) device
    Vp: object                 # (n_p, k_p) device
    W: object                  # (n, m) device collateral basis
    pi: np.ndarray             # (m,) EI rows (packed DOFs)
    arrays: dict               # device arrays of the hc_rom struct
    dims: dict
    struct: object = None

    @property
    def k(self) -> int:
        return self.k_c + self.k_p

    def host(self) -> dict:
        """numpy copies of the online data (for the CPU oracle)."""
        return {k: v.cpu().numpy() for k, v in self.arrays.items()} | dict(self.dims)

    def project(self, x):
        """x~ = B^T x."""
        t = _dev.torch()
        x = _dev.to_dev(x)
        nc = self.Vc.shape[0]
        return t.cat([tc_matmul(self.Vc.t(), x[:nc, None])[:, 0], tc_matmul(self.Vp.t(), x[nc:, None])[:, 0]])

    def lift(self, xt):
        """x = B x~ (reconstruction; not part of the online loop)."""
        t = _dev.torch()
        xt = _dev.to_dev(xt)
        return t.cat([tc_matmul(self.Vc, xt[: self.k_c, None])[:, 0], tc_matmul(self.Vp, xt[self.k_c:, None])[:, 0]])


def _face_tables(op):
    """Packed-DOF face lists of the operator (operator.py:246-327) as (kind, dofs[4], slot)
    plus the (row, face, coefficient) incidence of N."""
    tp = op.p.t_plus
    kinds, dofs, slots, inc = [], [], [], []
    f0 = 0

    def add(kind, cols, slot, rows_coefs):
        nonlocal f0
        nf = cols[0].size
        if not nf:
            return
        kinds.append(np.full(nf, kind, np.int32))
        d = np.full((nf, 4), -1, np.int64)
        for j, c in enumerate(cols):
            d[:, j] = c
        dofs.append(d)
        slots.append(np.asarray(slot, np.int64) if slot is not None else np.full(nf, -1, np.int64))
        fid = np.arange(f0, f0 + nf)
        for rows, coef in rows_coefs:
            inc.append((np.asarray(rows, np.int64), fid, np.full(nf, coef)))
        f0 += nf

    add(RF_BV, (op.bv_xc_gr, op.bv_xc_el, op.bv_xp_gr, op.bv_xp_el), None,
        [(op.bv_xc_gr, 1.0), (op.bv_xp_gr, 1.0), (op.bv_xc_el, -1.0), (op.bv_xp_el, -1.0)])
    add(RF_CE, (op.ce_xp_fo, op.ce_xc_el, op.ce_xp_el), None,
        [(op.ce_xp_fo, 1.0), (op.ce_xc_el, -1.0), (op.ce_xp_el, -1.0)])
    add(RF_STRIP, (op.strip_xp_pl, op.strip_xc_el, op.strip_xp_el), op.strip_slot,
        [(op.strip_xp_pl, 1.0), (op.strip_xc_el, -1.0), (op.strip_xp_el, -1.0)])
    add(RF_ELEL, (op.elel_xc_i, op.elel_xc_j, op.elel_xp_i, op.elel_xp_j), None,
        [(op.elel_xp_i, -1.0), (op.elel_xp_j, 1.0), (op.elel_xc_i, -tp), (op.elel_xc_j, tp)])
    cat = lambda xs, d: np.concatenate(xs) if xs else np.zeros(0, d)  # noqa: E731
    return (cat(kinds, np.int32), np.concatenate(dofs) if dofs else np.zeros((0, 4), np.int64),
            cat(slots, np.int64), cat([i[0] for i in inc], np.int64), cat([i[1] for i in inc], np.int64),
            cat([i[2] for i in inc], float))


def build_rom(op, snaps: Snapshots, k_c: int, k_p: int, m: int, rel_tol: float | None = None,
              separate_ei: bool = False, m_c: int | None = None) -> ReducedModel:
    """Offline stage: POD bases, EI data, projected blocks, restricted stencil.

    ``rel_tol`` truncates each POD basis by its discarded energy (ranks k_c, k_p are then
    upper bounds).  ``separate_ei`` interpolates the interface-current sub-operator A_bv
    (M = m points) and the chemical-potential sub-operator A_1/c (M = m_c, default m) in
    their own EI spaces, as SPEC build_rom's (M^(bv), M^(1/c)); the default is one EI space
    for their sum."""
    nc = op.dof.n_c
    Vc, _ = pod_rank(snaps.X[:nc], k_c, rel_tol)
    Vp, _ = pod_rank(snaps.X[nc:], k_p, rel_tol)
    if separate_ei:
        if snaps.Nb is None:
            raise ReductionError("separate EI spaces need the per-sub-operator snapshots")
        Wb, _ = pod_rank(snaps.Nb, m)
        Wc, _ = pod_rank(snaps.Nc, m_c or m)
        return assemble_rom(op, Vc, Vp, None, spaces=[(Wb, (RF_BV, RF_CE, RF_STRIP)), (Wc, (RF_ELEL,))])
    W, _ = pod_rank(snaps.N, m)
    return assemble_rom(op, Vc, Vp, W)


def build_rom_twin(op, snaps: Snapshots, k_c: int, k_p: int, m: int, keep_fraction: float = 0.97):
    """The reduced model and its validation twin (SPEC mor.build_rom, §3.2): the twin uses
    all k_c + k_p POD vectors and M^ = M + max(3, 3% of M) EI vectors, the model the first
    ceil(keep_fraction k) of each basis and the first M EI vectors — nested spaces, so
    their distance is measured in reduced coordinates."""
    import math
    nc = op.dof.n_c
    Vc, _ = pod_rank(snaps.X[:nc], k_c)
    Vp, _ = pod_rank(snaps.X[nc:], k_p)
    m_hat = m + max(3, int(math.ceil(0.03 * m)))
    W, _ = pod_rank(snaps.N, m_hat)
    twin = assemble_rom(op, Vc, Vp, W)
    kc = max(1, int(math.ceil(keep_fraction * Vc.shape[1])))
    kp = max(1, int(math.ceil(keep_fraction * Vp.shape[1])))
    rom = assemble_rom(op, Vc[:, :kc].contiguous(), Vp[:, :kp].contiguous(), W[:, :min(m, W.shape[1])].contiguous())
    return rom, twin


def assemble_rom(op, Vc, Vp, W, spaces=None) -> ReducedModel:
    """Projected blocks, EI rows / projection and the restricted stencil for given bases.

    ``spaces``: list of (collateral basis, face kinds) EI spaces; default one space W for
    all face kinds.  Each space contributes its DEIM rows (evaluated from its faces only)
    and its block of E = B^T W (W_pi)^-1."""
    t = _dev.torch()
    dof = op.dof
    nc, n = dof.n_c, dof.n_total
    k_c, k_p = Vc.shape[1], Vp.shape[1]
    k = k_c + k_p
    if k > 160:
        raise ReductionError("reduced dimension exceeds HC_ROM_MAX_K (160)")
    if spaces is None:
        spaces = [(W, (RF_BV, RF_CE, RF_STRIP, RF_ELEL))]
    pis = [deim(Ws) for Ws, _ in spaces]
    m = sum(Ws.shape[1] for Ws, _ in spaces)
    pi = np.concatenate(pis)
    # ---- affine blocks: A~ = B^T A_lin B, M~ = B^T diag(c rows) B, b~ = B^T b_bnd
    def Bcol(j):
        v = t.zeros(n, dtype=t.float64, device="cuda")
        if j < k_c:
            v[:nc] = Vc[:, j]
        else:
            v[nc:] = Vp[:, j - k_c]
        return v

    def BT(v):
        return t.cat([tc_matmul(Vc.t(), v[:nc, None])[:, 0], tc_matmul(Vp.t(), v[nc:, None])[:, 0]])

    A = t.stack([BT(op.apply_lin(Bcol(j))) for j in range(k)], dim=1)
    Mr = t.zeros((k, k), dtype=t.float64, device="cuda")
    Mr[:k_c, :k_c] = tc_matmul(Vc.t(), Vc)
    bnd = BT(_dev.to_dev(op.apply_bnd()))
    Es = []
    for (Ws, _), pis_ in zip(spaces, pis):
        Pi = t.as_tensor(pis_, device="cuda")
        BTW = t.cat([tc_matmul(Vc.t(), Ws[:nc]), tc_matmul(Vp.t(), Ws[nc:])])     # B^T W (DMMA)
        Es.append(t.linalg.solve(Ws[Pi].t(), BTW.t()).t())                       # B^T W (W_pi)^-1
    E = t.cat(Es, dim=1)
    v_cp, v_ac = qoi_vectors(dof)
    q_v, q_ac = BT(_dev.to_dev(v_cp)), BT(_dev.to_dev(v_ac))
    # ---- restricted stencil: faces of the EI rows + every stripping face
    kind, fdof, fslot, inc_row, inc_face, inc_coef = _face_tables(op)
    rms, rfs, rcs = [], [], []
    off = 0
    for (Ws, kinds), pis_ in zip(spaces, pis):   # each EI row reads its own space's faces
        row_of = np.full(n, -1, np.int64)
        row_of[pis_] = off + np.arange(pis_.size)
        sel = (row_of[inc_row] >= 0) & np.isin(kind[inc_face], kinds)
        rms.append(row_of[inc_row[sel]])
        rfs.append(inc_face[sel])
        rcs.append(inc_coef[sel])
        off += pis_.size
    r_m, r_f, r_c = np.concatenate(rms), np.concatenate(rfs), np.concatenate(rcs)
    active = np.union1d(np.unique(r_f), np.flatnonzero(kind == RF_STRIP))
    loc_face = np.full(kind.size, -1, np.int64)
    loc_face[active] = np.arange(active.size)
    adofs = fdof[active]
    S = np.unique(adofs[adofs >= 0])
    loc_dof = np.full(n, -1, np.int64)
    loc_dof[S] = np.arange(S.size)
    f_dof = np.where(adofs >= 0, loc_dof[np.maximum(adofs, 0)], -1).astype(np.int32)
    order = np.lexsort((loc_face[r_f], r_m))
    r_m, r_f, r_c = r_m[order], loc_face[r_f[order]], r_c[order]
    row_ptr = np.zeros(m + 1, np.int32)
    np.add.at(row_ptr, r_m + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.int32)
    a_kind, a_slot = kind[active], fslot[active]
    n_pl = int(dof.n_plated)
    strip_loc = np.flatnonzero(a_kind == RF_STRIP)
    strip_slot = a_slot[strip_loc]
    o = np.lexsort((strip_loc, strip_slot))
    pl_face = strip_loc[o].astype(np.int32)
    pl_ptr = np.zeros(max(n_pl, 0) + 1, np.int32)
    if n_pl:
        np.add.at(pl_ptr, strip_slot[o] + 1, 1)
        pl_ptr = np.cumsum(pl_ptr).astype(np.int32)
    Sd = t.as_tensor(S, device="cuda")
    BS = t.zeros((S.size, k), dtype=t.float64, device="cuda")
    isc = Sd < nc
    BS[isc, :k_c] = Vc[Sd[isc]]
    BS[~isc, k_c:] = Vp[Sd[~isc] - nc]
    dev = lambda a, dt=None: _dev.to_dev(a, dt)  # noqa: E731
    i32 = t.int32
    arrays = {
        "A": A.contiguous(), "Mr": Mr, "bnd": bnd, "E": E.contiguous(), "BS": BS,
        "f_kind": dev(a_kind.astype(np.int32), i32), "f_dof": dev(f_dof.reshape(-1), i32),
        "f_slot": dev(a_slot.astype(np.int32), i32), "row_ptr": dev(row_ptr, i32),
        "row_face": dev(r_f.astype(np.int32), i32), "row_coef": dev(r_c.astype(float)),
        "pl_ptr": dev(pl_ptr, i32), "pl_face": dev(pl_face if pl_face.size else np.zeros(1, np.int32), i32),
        "q_v": q_v, "q_ac": q_ac,
    }
    dims = {"k": k, "k_c": k_c, "m": m, "n_s": int(S.size), "n_f": int(active.size), "n_pl": n_pl}
    rom = ReducedModel(k_c, k_p, m, Vc, Vp, W, pi, arrays, dims)
    rom.struct = _native.HcRom(**dims, **{n_: _dev.ptr(a) for n_, a in arrays.items()})
    return rom


# ------------------------------------------------------------------ online
@dataclass
class RomTrajectory:
    xt: object                 # final reduced state (device)
    n_pl: object               # final plated inventory (device)
    voltage: np.ndarray        # per step
    mean_solid_c: np.ndarray   # per step
    newton_iters: np.ndarray
    states: object = None      # (n_steps, k) reduced states per step (device), if requested


def solve_rom(op, rom: ReducedModel, xt0, n_pl0, mu: float, dt: float, n_steps: int,
              rtol: float = 1e-10, max_iter: int = 40, refresh: int = 6,
              jac_steps: int = 8, keep_states: bool = False) -> RomTrajectory:
    """Reduced implicit-Euler trajectory, one kernel launch (hc_rom_run); the reduced
    Jacobian is refreshed every ``jac_steps`` steps (chord Newton in between)."""
    t = _dev.torch()
    xt = _dev.to_dev(xt0).clone()
    npl = _dev.to_dev(n_pl0 if _dev.numel(n_pl0) else np.zeros(1)).clone()
    qoi = t.empty(2 * max(n_steps, 1), dtype=t.float64, device="cuda")
    its = t.empty(max(n_steps, 1), dtype=t.int32, device="cuda")
    states = t.empty((max(n_steps, 1), rom.k), dtype=t.float64, device="cuda") if keep_states else None
    failed = ctypes.c_int32(-1)
    code = _native.lib().hc_rom_run(op.native.handle, ctypes.byref(rom.struct), _dev.ptr(xt),
                                    _dev.ptr(npl), float(mu), float(dt), int(n_steps), float(rtol),
                                    int(max_iter), int(refresh), int(jac_steps), _dev.ptr(qoi),
                                    _dev.ptr(its), _dev.ptr(states) if keep_states else None,
                                    ctypes.byref(failed), _dev.stream())
    if code:
        try:
            _native.check(code)
        except Exception as e:  # noqa: BLE001
            raise ReductionError(f"reduced Newton failed at step {failed.value}: {e}") from e
    q = qoi.cpu().numpy()[: 2 * n_steps].reshape(-1, 2) if n_steps else np.zeros((0, 2))
    return RomTrajectory(xt, npl, q[:, 0], q[:, 1], its.cpu().numpy()[:n_steps],
                         states[:n_steps] if keep_states else None)


def solve_rom_batch(op, rom: ReducedModel, xt0, n_pl0, mus, dt: float, n_steps: int,
                    rtol: float = 1e-10, max_iter: int = 40, refresh: int = 6, jac_steps: int = 8):
    """The reduced trajectory for many applied currents at once (the MOR use case): one
    thread-block cluster per value in a single launch (hc_rom_run_batch).  Returns
    (voltage (n_par, n_steps), mean solid c (n_par, n_steps), final x~ (n_par, k))."""
    t = _dev.torch()
    mus = np.asarray(mus, dtype=float)
    n_par = int(mus.size)
    xt = _dev.to_dev(xt0).reshape(1, -1).repeat(n_par, 1).contiguous()
    npl1 = np.asarray(n_pl0 if _dev.numel(n_pl0) else np.zeros(1), dtype=float)
    npl = _dev.to_dev(np.tile(npl1, (n_par, 1)))
    mu_d = _dev.to_dev(mus)
    qoi = t.empty((n_par, 2 * max(n_steps, 1)), dtype=t.float64, device="cuda")
    its = t.empty((n_par, max(n_steps, 1)), dtype=t.int32, device="cuda")
    failed = (ctypes.c_int32 * n_par)()
    code = _native.lib().hc_rom_run_batch(op.native.handle, ctypes.byref(rom.struct), n_par, _dev.ptr(xt),
                                          _dev.ptr(npl), _dev.ptr(mu_d), float(dt), int(n_steps), float(rtol),
                                          int(max_iter), int(refresh), int(jac_steps), _dev.ptr(qoi),
                                          _dev.ptr(its), failed, _dev.stream())
    if code:
        bad = [(i, f) for i, f in enumerate(failed) if f >= 0]
        try:
            _native.check(code)
        except Exception as e:  # noqa: BLE001
            raise ReductionError(f"reduced Newton failed for (parameter, step) {bad[:4]}: {e}") from e
    q = qoi.cpu().numpy()[:, : 2 * n_steps].reshape(n_par, -1, 2)
    return q[..., 0], q[..., 1], xt


def estimate_error(op, rom: ReducedModel, twin: ReducedModel, x0, n_pl0, mu: float, dt: float,
                   n_steps: int, theta: float = 0.0, **kw):
    """Hierarchical error estimate (SPEC mor.estimate_error; arXiv 1704.04139 Eqs. 21-22):
    run the model and its (nested, larger) validation twin and return, per field,
    1/(1-theta) max_n ||x~_n - x^_n|| / ||x^_n||  (L-infinity in time of relative L2 in
    space), evaluated in the twin's reduced coordinates — exact because the bases are
    nested and orthonormal."""
    if not 0.0 <= theta < 1.0:
        raise ValueError("theta must be in [0, 1)")
    t = _dev.torch()
    a = solve_rom(op, rom, rom.project(x0), n_pl0, mu, dt, n_steps, keep_states=True, **kw)
    b = solve_rom(op, twin, twin.project(x0), n_pl0, mu, dt, n_steps, keep_states=True, **kw)
    sa, sb = a.states, b.states
    kc, kc2 = rom.k_c, twin.k_c
    dc = sb[:, :kc2].clone()
    dc[:, :kc] -= sa[:, :kc]
    dp = sb[:, kc2:].clone()
    dp[:, : rom.k_p] -= sa[:, kc:]
    rel = lambda d, ref: float(t.max(t.linalg.vector_norm(d, dim=1) / t.linalg.vector_norm(ref, dim=1)))  # noqa: E731
    f = 1.0 / (1.0 - theta)
    return f * rel(dc, sb[:, :kc2]), f * rel(dp, sb[:, kc2:])
