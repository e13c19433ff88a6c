"""Full and restricted access to the nonlinear sub-operators, for empirical interpolation.

Drop-in for ``SubOperatorView`` / ``RestrictedSubOperator`` of the reference
(``src/halfcell/fvm/operator.py:476-646``): ``op.sub_operator("bv" | "one_over_c")``
gives the view (``dim``, ``apply``, ``output_dofs``, ``source_dofs``,
``restricted``); ``view.restricted(rows)`` evaluates the selected output rows, and
their local Jacobian, from the stencil DOF values only.

The restricted evaluation runs on the GPU (``hc_restricted_eval``) from the same
face table — kinds, stencil positions, plated slots, (row, face, coefficient)
incidence — and the same face-kinetics device function that the reduced model's
online kernel (``csrc/hc_rom.cu``) evaluates its EI rows with, so checking it
against the reference's ``RestrictedSubOperator`` pins the ROM's EI evaluation.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _native

RF_BV, RF_CE, RF_STRIP, RF_ELEL = 0, 1, 2, 3
_FAMILY_KINDS = {"bv": (RF_BV, RF_CE, RF_STRIP), "one_over_c": (RF_ELEL,)}
# face-table columns (stencil positions) each kind reads, operator.py:498-513 col arrays:
# BV (c_gr, c_el, phi_gr, phi_el); CE (phi_fo, -, phi_el); STRIP (phi_pl, c_el, phi_el);
# ELEL (c_i, c_j, -, -)
_READS = {RF_BV: (0, 1, 2, 3), RF_CE: (0, 2), RF_STRIP: (0, 1, 2), RF_ELEL: (0, 1)}


def face_tables(op):
    """(kind, dofs[n_f, 4], slot, inc_row, inc_face, inc_coef) of every interface /
    electrolyte face of ``op`` in the reference's family order (mor._face_tables)."""
    from .mor import _face_tables
    return _face_tables(op)


class SubOperatorView:
    """Uniform full/restricted access to one nonlinear sub-operator (operator.py:482-538)."""

    def __init__(self, op, which: str):
        if which not in _FAMILY_KINDS:
            raise KeyError(which)
        self.op = op
        self.which = which

    @property
    def dim(self) -> int:
        return self.op.dof.n_total

    def apply(self, x, n_pl, beta: float = 0.0):
        if self.which == "bv":
            return self.op.apply_bv(x, n_pl, beta=beta)
        return self.op.apply_one_over_c(x)

    def _tables(self):
        if not hasattr(self, "_tab"):
            kind, dofs, slot, inc_row, inc_face, inc_coef = face_tables(self.op)
            keep_f = np.isin(kind, _FAMILY_KINDS[self.which])
            keep_i = keep_f[inc_face] if inc_face.size else np.zeros(0, bool)
            self._tab = (kind, dofs, slot, inc_row[keep_i], inc_face[keep_i], inc_coef[keep_i])
        return self._tab

    def output_dofs(self) -> np.ndarray:
        _, _, _, inc_row, _, _ = self._tables()
        return np.unique(inc_row) if inc_row.size else np.empty(0, dtype=np.int64)

    def _touched_faces(self, out_rows: np.ndarray) -> np.ndarray:
        _, _, _, inc_row, inc_face, _ = self._tables()
        return np.unique(inc_face[np.isin(inc_row, out_rows)])

    def source_dofs(self, out_rows) -> np.ndarray:
        """Input DOFs needed to evaluate the sub-operator at ``out_rows`` (operator.py:524-535)."""
        out_rows = np.unique(np.asarray(out_rows, dtype=np.int64))
        kind, dofs, _, _, _, _ = self._tables()
        faces = self._touched_faces(out_rows)
        need = [dofs[faces[kind[faces] == k]][:, list(cols)].ravel() for k, cols in _READS.items()]
        need = np.concatenate(need) if need else np.empty(0, np.int64)
        return np.unique(need[need >= 0]) if need.size else np.empty(0, dtype=np.int64)

    def restricted(self, out_rows) -> "RestrictedSubOperator":
        return RestrictedSubOperator(self, np.unique(np.asarray(out_rows, dtype=np.int64)))


class RestrictedSubOperator:
    """Selected output rows of a sub-operator from a small stencil (operator.py:541-646).

    ``rows`` are the (sorted, unique) output DOFs, ``stencil`` the state DOFs they
    depend on; :meth:`apply` / :meth:`jacobian` take the stencil values ``x_st`` and
    never touch a full-order-length array (all index work is done here, once).
    """

    def __init__(self, view: SubOperatorView, out_rows: np.ndarray):
        self.view = view
        self.op = view.op
        self.rows = out_rows
        self.stencil = view.source_dofs(out_rows)
        kind, dofs, slot, inc_row, inc_face, inc_coef = view._tables()
        sel = np.isin(inc_row, out_rows)
        r_row = np.searchsorted(out_rows, inc_row[sel])
        faces = np.unique(inc_face[sel])
        loc_face = np.full(kind.size, -1, np.int64)
        loc_face[faces] = np.arange(faces.size)
        r_face = loc_face[inc_face[sel]]
        order = np.lexsort((r_face, r_row))
        r_row, r_face, r_coef = r_row[order], r_face[order], inc_coef[sel][order]
        row_ptr = np.zeros(out_rows.size + 1, np.int64)
        np.add.at(row_ptr, r_row + 1, 1)
        row_ptr = np.cumsum(row_ptr)
        fk = kind[faces]
        fd = np.full((faces.size, 4), -1, np.int64)
        for k, cols in _READS.items():
            m = fk == k
            for c in cols:
                fd[m, c] = np.searchsorted(self.stencil, dofs[faces[m], c])
        t = _dev.torch()
        i32 = t.int32
        self._n_f = int(faces.size)
        self._arr = {
            "f_kind": _dev.to_dev(fk.astype(np.int32), i32),
            "f_dof": _dev.to_dev(fd.reshape(-1).astype(np.int32), i32),
            "f_slot": _dev.to_dev(slot[faces].astype(np.int32), i32),
            "row_ptr": _dev.to_dev(row_ptr.astype(np.int32), i32),
            "row_face": _dev.to_dev(r_face.astype(np.int32), i32),
            "row_coef": _dev.to_dev(r_coef.astype(np.float64)),
        }

    def _eval(self, x_st, n_pl, beta: float, want_jac: bool):
        a = self._arr
        xs = _dev.to_dev(x_st)
        npl = _dev.to_dev(n_pl if _dev.numel(n_pl) else np.zeros(1))
        out = _dev.empty(self.rows.size)
        jac = _dev.empty(self.rows.size * self.stencil.size) if want_jac else None
        _native.check(_native.lib().hc_restricted_eval(
            self.op.native.handle, int(self.rows.size), self._n_f, int(self.stencil.size),
            _dev.ptr(a["f_kind"]), _dev.ptr(a["f_dof"]), _dev.ptr(a["f_slot"]), _dev.ptr(a["row_ptr"]),
            _dev.ptr(a["row_face"]), _dev.ptr(a["row_coef"]), _dev.ptr(xs), _dev.ptr(npl), float(beta),
            _dev.ptr(out), _dev.ptr(jac) if want_jac else None, _dev.stream()))
        return out, jac

    def apply(self, x_st, n_pl, beta: float = 0.0):
        """Selected-row values; ``x_st`` holds the stencil DOF values."""
        out, _ = self._eval(x_st, n_pl, beta, False)
        return _dev.like_input(out, x_st)

    def jacobian(self, x_st, n_pl, beta: float = 0.0):
        """Local Jacobian (selected rows x stencil DOFs) as ``scipy.sparse.csr_matrix``."""
        import scipy.sparse as sp
        _, jac = self._eval(x_st, n_pl, beta, True)
        dense = jac.reshape(self.rows.size, self.stencil.size).cpu().numpy()
        return sp.csr_matrix(dense)
