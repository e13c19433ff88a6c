"""ctypes binding of ``libhalfcell_b200.so`` (the C ABI in ``include/halfcell_b200.h``).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises :class:`NativeError`.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (ConfigError, HalfcellError, ModelError, NativeError, NonConvergence,
                     NumericsError, ReductionError, SimulationError)
from .params import HcParams

LIB_PATH = os.environ.get("HC_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhalfcell_b200.so")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int64_p = ctypes.POINTER(ctypes.c_int64)


class HcInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "nx", "ny", "nz", "n_vox", "n_c", "n_p", "n_plated", "n_dirichlet",
        "n_bv", "n_ce", "n_strip", "n_elel", "n_drive_faces")] + [
        (n, ctypes.c_double) for n in ("h", "face_area", "voxel_volume", "n_const", "scale")]


class HcSolverConfig(ctypes.Structure):
    _fields_ = [("newton_rtol", ctypes.c_double), ("newton_atol", ctypes.c_double),
                ("newton_max_iter", ctypes.c_int32), ("krylov_max_iter", ctypes.c_int32),
                ("linear_rtol", ctypes.c_double), ("dt_init", ctypes.c_double),
                ("dt_min", ctypes.c_double), ("dt_max", ctypes.c_double),
                ("grow_factor", ctypes.c_double), ("shrink_factor", ctypes.c_double),
                ("easy_iter_threshold", ctypes.c_int32), ("implicit_plated", ctypes.c_int32),
                ("linear_safety", ctypes.c_double)]


class HcNewtonStats(ctypes.Structure):
    _fields_ = [("n_iter", ctypes.c_int32), ("krylov_iters", ctypes.c_int32),
                ("retries", ctypes.c_int32), ("status", ctypes.c_int32),
                ("norm0", ctypes.c_double), ("norm_final", ctypes.c_double),
                ("tol", ctypes.c_double), ("dt_used", ctypes.c_double),
                ("dt_next", ctypes.c_double), ("clamped_loss", ctypes.c_double)]


class HcRom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("k", "k_c", "m", "n_s", "n_f", "n_pl")] + [
        (n, ctypes.c_void_p) for n in ("A", "Mr", "bnd", "E", "BS", "f_kind", "f_dof", "f_slot",
                                       "row_ptr", "row_face", "row_coef", "pl_ptr", "pl_face",
                                       "q_v", "q_ac")]


_ERRORS = {1: NativeError, 2: ModelError, 3: NumericsError, 4: NonConvergence,
           5: ConfigError, 6: SimulationError, 7: ReductionError}

_lib = None

_SIGS = {
    "hc_last_error": (ctypes.c_char_p, []),
    "hc_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "hc_operator_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_double,
                                          ctypes.POINTER(HcParams),
                                          ctypes.POINTER(ctypes.c_void_p)]),
    "hc_operator_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "hc_operator_set_params": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "hc_operator_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(HcInfo)]),
    "hc_operator_export": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "hc_apply": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_double, ctypes.c_double, ctypes.c_void_p,
                                ctypes.c_void_p]),
    "hc_jvp": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                              ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "hc_jacobian_csr": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_double, c_int64_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "hc_newton_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                       ctypes.POINTER(HcSolverConfig), ctypes.c_void_p,
                                       ctypes.POINTER(HcNewtonStats), ctypes.c_void_p]),
    "hc_solve_initial_potential": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                                  ctypes.c_void_p, ctypes.c_double,
                                                  ctypes.POINTER(HcSolverConfig),
                                                  ctypes.c_void_p, ctypes.POINTER(HcNewtonStats),
                                                  ctypes.c_void_p]),
    "hc_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                               ctypes.c_double, ctypes.c_double, ctypes.POINTER(HcSolverConfig),
                               ctypes.POINTER(HcNewtonStats), ctypes.c_void_p]),
    "hc_step_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.POINTER(HcSolverConfig),
                                    ctypes.POINTER(HcNewtonStats)]),
    "hc_lin_csr": (ctypes.c_int, [ctypes.c_void_p, c_int64_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p]),
    "hc_strip_face_currents": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]),
    "hc_restricted_eval": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32] + [ctypes.c_void_p] * 8
                           + [ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "hc_newton_solve_ex": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                          ctypes.POINTER(HcSolverConfig), ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                          ctypes.c_int32, ctypes.c_void_p,
                                          ctypes.POINTER(HcNewtonStats), ctypes.c_void_p]),
    "hc_step_ex": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                  ctypes.c_double, ctypes.c_double, ctypes.POINTER(HcSolverConfig),
                                  ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(HcNewtonStats),
                                  ctypes.c_void_p]),
    "hc_precond_refresh": (ctypes.c_int, [ctypes.c_void_p]),
    "hc_dgemm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                ctypes.c_void_p]),
    "hc_dmma_peak": (ctypes.c_int, [c_double_p, ctypes.c_void_p]),
    "hc_launch_count": (ctypes.c_int, [c_int64_p]),
    "hc_flush_l2": (ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p]),
    "hc_time_kernels": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "hc_step_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.POINTER(HcSolverConfig), ctypes.c_void_p,
                                     ctypes.c_int32]),
    "hc_pod_gram": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                   ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "hc_pod_gram_rows": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "hc_rom_run_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(HcRom), ctypes.c_int32,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                        ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]),
    "hc_rom_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(HcRom), ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                  ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.POINTER(ctypes.c_int32), ctypes.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare every exported signature."""
    if not os.path.exists(path):
        raise NativeError(f"CUDA library {path} is missing; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def check(code: int) -> None:
    if code != 0:
        msg = lib().hc_last_error().decode(errors="replace")
        raise _ERRORS.get(code, HalfcellError)(msg)


def require_device() -> None:
    n = ctypes.c_int(0)
    check(lib().hc_device_count(ctypes.byref(n)))
    if n.value < 1:
        raise NativeError("no CUDA device visible; the halfcell_b200 path runs only on the GPU")
