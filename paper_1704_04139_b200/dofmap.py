"""DOF layout on a phase grid, numbered on the GPU.

Mirrors ``halfcell.fvm.dofmap`` (reference ``src/halfcell/fvm/dofmap.py:20-101``):
c DOFs on graphite and electrolyte voxels, phi DOFs on every voxel except the
grounded counter-collector voxels of the outermost z layer, packed state
``x = [c-block, phi-block]``.  Validation (missing phases, no electrolyte path,
no counter collector to ground) runs in the CUDA library and raises the same
``ModelError`` messages.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .params import MaterialParams, to_c_params
from .phases import PhaseGrid


class NativeOperator:
    """Owner of one ``hc_operator`` handle (device-resident geometry + work space)."""

    def __init__(self, grid: PhaseGrid, params: MaterialParams):
        _native.require_device()
        L = _native.lib()
        nz, ny, nx = grid.labels.shape
        labels = np.ascontiguousarray(grid.labels, dtype=np.uint8)
        self._cp = to_c_params(params)
        h = ctypes.c_void_p()
        _native.check(L.hc_operator_create(labels.ctypes.data, nx, ny, nz, float(grid.voxel_size),
                                           ctypes.byref(self._cp), ctypes.byref(h)))
        self.handle = h
        info = _native.HcInfo()
        _native.check(L.hc_operator_info(h, ctypes.byref(info)))
        self.info = info

    def set_params(self, params: MaterialParams) -> None:
        """New material parameters on the same classified geometry (``hc_operator_set_params``)."""
        cp = to_c_params(params)
        _native.check(_native.lib().hc_operator_set_params(self.handle, ctypes.byref(cp)))
        self._cp = cp
        _native.check(_native.lib().hc_operator_info(self.handle, ctypes.byref(self.info)))

    def export(self, what: int, length: int) -> np.ndarray:
        out = np.empty(max(length, 0), dtype=np.int64)
        if length:
            _native.check(_native.lib().hc_operator_export(self.handle, what, out.ctypes.data))
        return out

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            _native.lib().hc_operator_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Dofmap:
    grid: PhaseGrid
    c_dof: np.ndarray
    p_dof: np.ndarray
    n_c: int
    n_p: int
    plated_voxels: np.ndarray
    dirichlet: np.ndarray
    # the device operator build_dofmap classified the geometry with; the first SystemOperator
    # built on this Dofmap takes it over (new parameters, same geometry) instead of
    # classifying the grid a second time
    _nat: "NativeOperator | None" = field(default=None, init=False, repr=False, compare=False)

    def take_native(self) -> "NativeOperator | None":
        nat, self._nat = self._nat, None
        return nat

    @property
    def n_total(self) -> int:
        return self.n_c + self.n_p

    @property
    def n_plated(self) -> int:
        return int(self.plated_voxels.size)

    def x_index_c(self, voxel_flat) -> np.ndarray:
        return self.c_dof[voxel_flat]

    def x_index_p(self, voxel_flat) -> np.ndarray:
        return self.n_c + self.p_dof[voxel_flat]

    def voxel_coords(self, voxel_flat: int) -> tuple[int, int, int]:
        nz, ny, nx = self.grid.shape
        z, rem = divmod(int(voxel_flat), ny * nx)
        y, x = divmod(rem, nx)
        return x, y, z

    def describe(self) -> str:
        return (f"{self.n_c} concentration DOFs, {self.n_p} potential DOFs, "
                f"{self.n_plated} plated voxels, {self.dirichlet.size} grounded voxels")


def dofmap_from_native(grid: PhaseGrid, nat: NativeOperator) -> Dofmap:
    info = nat.info
    n = int(info.n_vox)
    return Dofmap(grid, nat.export(0, n), nat.export(1, n), int(info.n_c), int(info.n_p),
                  nat.export(2, int(info.n_plated)), nat.export(3, int(info.n_dirichlet)))


def build_dofmap(grid: PhaseGrid) -> Dofmap:
    """Number the DOFs and validate the grid (reference ``dofmap.py:71-101``)."""
    nat = NativeOperator(grid, MaterialParams())
    try:
        dof = dofmap_from_native(grid, nat)
    except BaseException:
        nat.close()
        raise
    dof._nat = nat
    return dof
