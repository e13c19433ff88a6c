"""Cell-centred finite-volume operator on the voxel grid, evaluated by CUDA kernels.

Drop-in for ``halfcell.fvm.operator`` (reference ``src/halfcell/fvm/operator.py``):
same constructor ``SystemOperator(dofmap, params)``, same attribute names for
the face lists and coefficients, same ``apply*`` decomposition

    A(x; mu) = b_const + mu * b_bnd + A_lin x + A_bv(x) + A_1c(x)

(``operator.py:9-18``) and the same sign conventions.  Inputs may be numpy
arrays (copied to the device, result returned as numpy) or CUDA fp64 tensors
(result stays on the device).  :meth:`jacobian` returns the reference's
``scipy.sparse.csr_matrix`` (assembled from the device linearization, for API and
sparsity parity); the solver path never assembles it and applies the Jacobian
matrix-free instead (:meth:`jvp`, :meth:`jacobian_operator`).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _dev, _native
from .dofmap import Dofmap, NativeOperator
from .errors import ModelError
from .params import MaterialParams

_PART = {"apply": 0, "bv": 1, "one_over_c": 2, "lin": 3, "const": 4, "bnd": 5}


@dataclass
class BoundaryDrive:
    """Applied current density (A/m^2) on the working-collector outer face (operator.py:55-67)."""

    mu: float = 0.0

    def __post_init__(self):
        if not np.isfinite(self.mu):
            raise ModelError("applied current density must be finite")


class JacobianOperator:
    """Matrix-free ``jacobian(x) + diag(mass)`` at a fixed state."""

    def __init__(self, op: "SystemOperator", x, n_pl, beta: float, inv_dt: float = 0.0):
        self.op, self.x, self.n_pl, self.beta, self.inv_dt = op, x, n_pl, beta, inv_dt
        self.shape = (op.dof.n_total, op.dof.n_total)

    def __matmul__(self, v):
        return self.op.jvp(self.x, self.n_pl, v, beta=self.beta, inv_dt=self.inv_dt)

    matvec = __matmul__

    def tocsr(self):
        return self.op.jacobian_csr(self.x, self.n_pl, beta=self.beta)


class SystemOperator:
    """Device-resident FV operator with the reference's exact decomposition."""

    def __init__(self, dofmap: Dofmap, params: MaterialParams):
        self.dof = dofmap
        self.p = params
        self.h = dofmap.grid.voxel_size * 1e-6
        self.face_area = self.h ** 2
        self.voxel_volume = self.h ** 3
        self.n_const = params.n_const(self.face_area)
        self._scale = 1.0 / (params.constants.F * self.h)
        nat = dofmap.take_native()
        if nat is not None:
            nat.set_params(params)   # same geometry: no second classification pass
            self.native = nat
        else:
            self.native = NativeOperator(dofmap.grid, params)
        info = self.native.info
        if int(info.n_c) != dofmap.n_c or int(info.n_p) != dofmap.n_p:
            raise ModelError("dofmap does not belong to this grid")
        F = params.constants.F
        self.gX = (params.kappa_el * (params.t_plus - 1.0) * params.constants.R
                   * params.temperature * (1.0 + params.dlnf_dlnc)) / (F ** 2 * self.h ** 2)
        self.n_drive_faces = int(info.n_drive_faces)
        self.drive_area = self.n_drive_faces * self.face_area
        self._lists = {}

    # --- face lists in the reference layout (operator.py:186-219) ----------------
    def _family(self, what: int, n: int, k: int) -> np.ndarray:
        if what not in self._lists:
            self._lists[what] = self.native.export(what, n * k).reshape(k, n)
        return self._lists[what]

    @property
    def n_bv(self) -> int:
        return int(self.native.info.n_bv)

    def _bv(self, i):
        return self._family(4, self.n_bv, 4)[i]

    def _ce(self, i):
        return self._family(5, int(self.native.info.n_ce), 3)[i]

    def _st(self, i):
        return self._family(6, int(self.native.info.n_strip), 4)[i]

    def _el(self, i):
        return self._family(7, int(self.native.info.n_elel), 4)[i]

    bv_xc_gr = property(lambda s: s._bv(0))
    bv_xc_el = property(lambda s: s._bv(1))
    bv_xp_gr = property(lambda s: s._bv(2))
    bv_xp_el = property(lambda s: s._bv(3))
    ce_xp_fo = property(lambda s: s._ce(0))
    ce_xc_el = property(lambda s: s._ce(1))
    ce_xp_el = property(lambda s: s._ce(2))
    strip_xp_pl = property(lambda s: s._st(0))
    strip_xc_el = property(lambda s: s._st(1))
    strip_xp_el = property(lambda s: s._st(2))
    strip_slot = property(lambda s: s._st(3))
    elel_xc_i = property(lambda s: s._el(0))
    elel_xc_j = property(lambda s: s._el(1))
    elel_xp_i = property(lambda s: s._el(2))
    elel_xp_j = property(lambda s: s._el(3))

    # --- evaluations -----------------------------------------------------------
    def _apply_part(self, part: str, x, n_pl, mu: float = 0.0, beta: float = 0.0):
        n = self.dof.n_total
        xd = _dev.to_dev(x) if x is not None else _dev.to_dev(np.ones(n))
        nd = _dev.to_dev(n_pl) if n_pl is not None else _dev.to_dev(
            np.zeros(max(self.dof.n_plated, 1)))
        out = _dev.empty(n)
        _native.check(_native.lib().hc_apply(self.native.handle, _PART[part], _dev.ptr(xd),
                                             _dev.ptr(nd), float(mu), float(beta),
                                             _dev.ptr(out), _dev.stream()))
        return _dev.like_input(out, x)

    def apply(self, x, n_pl, mu: float, beta: float = 0.0):
        """Full space operator A_mu(x) (operator.py:381-389); NumericsError on non-finite rows."""
        return self._apply_part("apply", x, n_pl, mu, beta)

    def apply_bv(self, x, n_pl, beta: float = 0.0):
        return self._apply_part("bv", x, n_pl, 0.0, beta)

    def apply_one_over_c(self, x):
        return self._apply_part("one_over_c", x, None)

    def apply_lin(self, x):
        return self._apply_part("lin", x, None)

    def apply_const(self, x=None):
        return np.zeros(self.dof.n_total)

    def apply_bnd(self, x=None):
        return self._apply_part("bnd", None, None) if x is None else self._apply_part("bnd", x, None)

    @property
    def b_const(self) -> np.ndarray:
        return np.zeros(self.dof.n_total)

    @property
    def b_bnd(self) -> np.ndarray:
        return np.asarray(self.apply_bnd())

    def jvp(self, x, n_pl, v, beta: float = 0.0, inv_dt: float = 0.0):
        """(jacobian(x) + diag(inv_dt on c rows)) @ v, matrix-free on the GPU."""
        xd, vd = _dev.to_dev(x), _dev.to_dev(v)
        nd = _dev.to_dev(n_pl) if n_pl is not None and _dev.numel(n_pl) else _dev.to_dev(np.zeros(1))
        out = _dev.empty(self.dof.n_total)
        _native.check(_native.lib().hc_jvp(self.native.handle, _dev.ptr(xd), _dev.ptr(nd),
                                           float(beta), float(inv_dt), _dev.ptr(vd),
                                           _dev.ptr(out), _dev.stream()))
        return _dev.like_input(out, v)

    def jacobian(self, x, n_pl, mu: float = 0.0, beta: float = 0.0):
        """Analytic Jacobian of :meth:`apply` as ``scipy.sparse.csr_matrix``
        (operator.py:458-471: A_lin + J_nl, duplicates summed, exact zeros dropped)."""
        return self.jacobian_csr(x, n_pl, beta=beta)

    def jacobian_operator(self, x, n_pl, beta: float = 0.0, inv_dt: float = 0.0) -> JacobianOperator:
        """``jacobian(x) + diag(inv_dt on c rows)`` as a matrix-free operator on the GPU."""
        return JacobianOperator(self, x, n_pl, beta, inv_dt)

    @property
    def A_lin(self):
        """The affine part's matrix (operator.py:221) as ``scipy.sparse.csr_matrix``."""
        if "A_lin" not in self._lists:
            import scipy.sparse as sp
            L = _native.lib()
            nnz = ctypes.c_int64(0)
            _native.check(L.hc_lin_csr(self.native.handle, ctypes.byref(nnz), None, None, None))
            n = self.dof.n_total
            rp = np.empty(n + 1, dtype=np.int64)
            ci = np.empty(nnz.value, dtype=np.int64)
            va = np.empty(nnz.value, dtype=np.float64)
            _native.check(L.hc_lin_csr(self.native.handle, ctypes.byref(nnz), rp.ctypes.data,
                                       ci.ctypes.data, va.ctypes.data))
            self._lists["A_lin"] = sp.csr_matrix((va, ci, rp), shape=(n, n))
        return self._lists["A_lin"]

    def strip_face_currents(self, x, n_pl, beta: float = 0.0):
        """(stripping current A/m^2, plated slot) for every stripping face (operator.py:391-399)."""
        slots = self.strip_slot
        if slots.size == 0:
            return (_dev.empty(0) if _dev.is_tensor(x) else np.empty(0)), slots
        xd = _dev.to_dev(x)
        nd = _dev.to_dev(n_pl)
        out = _dev.empty(slots.size)
        _native.check(_native.lib().hc_strip_face_currents(self.native.handle, _dev.ptr(xd), _dev.ptr(nd),
                                                           float(beta), _dev.ptr(out), _dev.stream()))
        return _dev.like_input(out, x), slots

    def sub_operator(self, name: str):
        """Uniform full / restricted access to one nonlinear sub-operator (operator.py:476-479)."""
        from .suboperator import SubOperatorView
        if name not in ("bv", "one_over_c"):
            raise KeyError(name)
        return SubOperatorView(self, name)

    def jacobian_csr(self, x, n_pl, beta: float = 0.0):
        import scipy.sparse as sp
        xd = _dev.to_dev(x)
        nd = _dev.to_dev(n_pl) if n_pl is not None and _dev.numel(n_pl) else _dev.to_dev(np.zeros(1))
        L = _native.lib()
        nnz = ctypes.c_int64(0)
        _native.check(L.hc_jacobian_csr(self.native.handle, _dev.ptr(xd), _dev.ptr(nd),
                                        float(beta), ctypes.byref(nnz), None, None, None))
        n = self.dof.n_total
        rp = np.empty(n + 1, dtype=np.int64)
        ci = np.empty(nnz.value, dtype=np.int64)
        va = np.empty(nnz.value, dtype=np.float64)
        _native.check(L.hc_jacobian_csr(self.native.handle, _dev.ptr(xd), _dev.ptr(nd),
                                        float(beta), ctypes.byref(nnz), rp.ctypes.data,
                                        ci.ctypes.data, va.ctypes.data))
        return sp.csr_matrix((va, ci, rp), shape=(n, n))
