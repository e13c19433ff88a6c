"""Physical constants and material parameters.

Same fields, defaults, units and validation as the reference
``src/halfcell/echem/params.py:20-129`` so a ``MaterialParams`` built for the
reference can be handed over field by field (see :func:`from_reference`).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field, fields

import numpy as np

from .errors import ConfigError

FARADAY = 96485.33
GAS_CONSTANT = 8.3145


@dataclass(frozen=True)
class PhysConstants:
    F: float = FARADAY
    R: float = GAS_CONSTANT


#: Synthetic graphite OCP table (SOC, volts); reference ``params.py:34-47``.
DEFAULT_OCP_TABLE = (
    (0.00, 0.600), (0.04, 0.400), (0.10, 0.280), (0.20, 0.220),
    (0.30, 0.210), (0.45, 0.185), (0.55, 0.155), (0.65, 0.150),
    (0.80, 0.145), (0.90, 0.100), (0.97, 0.070), (1.00, 0.060),
)

_POSITIVE = ("temperature", "d_gr", "sigma_gr", "sigma_li", "sigma_cc", "sigma_pl",
             "d_el", "kappa_el", "i00_grel", "i00_ceel", "i00_plel", "c_gr_max",
             "n_const_thickness", "c_li_metal", "c_el_init")


@dataclass
class MaterialParams:
    """Transport and kinetic coefficients, SI units (reference ``params.py:50-113``)."""

    temperature: float = 298.15
    d_gr: float = 5.0e-13
    sigma_gr: float = 50.0
    sigma_li: float = 2.0e3
    sigma_cc: float = 2.0e3
    sigma_pl: float = 2.0e3
    d_el: float = 3.0e-10
    kappa_el: float = 1.0
    t_plus: float = 0.26
    dlnf_dlnc: float = 0.0
    i00_grel: float = 2.0e-4
    i00_ceel: float = 50.0
    i00_plel: float = 2.0
    c_gr_max: float = 30000.0
    ocp_table: tuple = DEFAULT_OCP_TABLE
    n_const_thickness: float = 0.48e-9
    c_li_metal: float = 76900.0
    c_el_init: float = 1000.0
    soc_init: float = 0.75
    constants: PhysConstants = field(default_factory=PhysConstants)

    def __post_init__(self):
        self.validate()

    def validate(self):
        for name in _POSITIVE:
            if getattr(self, name) <= 0:
                raise ConfigError(f"{name} must be positive")
        if not 0.0 < self.t_plus < 1.0:
            raise ConfigError("transference number must lie in (0, 1)")
        if not 0.0 < self.soc_init <= 1.0:
            raise ConfigError("initial state of charge must lie in (0, 1]")
        socs = [s for s, _ in self.ocp_table]
        if len(socs) < 2 or socs[0] > 0.0 or socs[-1] < 1.0:
            raise ConfigError("OCP table must cover SOC in [0, 1]")
        if any(b <= a for a, b in zip(socs, socs[1:])):
            raise ConfigError("OCP table SOC knots must be strictly increasing")
        if len(socs) > HC_MAX_OCP:
            raise ConfigError(f"OCP table is limited to {HC_MAX_OCP} knots on the device")

    def n_const(self, face_area: float) -> float:
        """Regularization inventory (mol) of one voxel face, reference ``params.py:102-108``."""
        return self.c_li_metal * self.n_const_thickness * face_area

    @property
    def thermal_voltage_2(self) -> float:
        """2 R T / F (reference ``params.py:110-113``)."""
        return 2.0 * self.constants.R * self.temperature / self.constants.F

    @classmethod
    def from_reference(cls, ref) -> "MaterialParams":
        """Copy every field of a reference ``halfcell.echem.MaterialParams``."""
        kw = {f.name: getattr(ref, f.name) for f in fields(cls) if f.name != "constants"}
        kw["constants"] = PhysConstants(ref.constants.F, ref.constants.R)
        return cls(**kw)


HC_MAX_OCP = 32


class HcParams(ctypes.Structure):
    """C mirror of ``hc_params`` in ``include/halfcell_b200.h``."""

    _fields_ = [
        ("temperature", ctypes.c_double), ("d_gr", ctypes.c_double),
        ("sigma_gr", ctypes.c_double), ("sigma_li", ctypes.c_double),
        ("sigma_cc", ctypes.c_double), ("sigma_pl", ctypes.c_double),
        ("d_el", ctypes.c_double), ("kappa_el", ctypes.c_double),
        ("t_plus", ctypes.c_double), ("dlnf_dlnc", ctypes.c_double),
        ("i00_grel", ctypes.c_double), ("i00_ceel", ctypes.c_double),
        ("i00_plel", ctypes.c_double), ("c_gr_max", ctypes.c_double),
        ("n_const_thickness", ctypes.c_double), ("c_li_metal", ctypes.c_double),
        ("faraday", ctypes.c_double), ("gas_constant", ctypes.c_double),
        ("n_ocp", ctypes.c_int32), ("pad_", ctypes.c_int32),
        ("ocp_soc", ctypes.c_double * HC_MAX_OCP), ("ocp_v", ctypes.c_double * HC_MAX_OCP),
    ]


def to_c_params(p: MaterialParams) -> HcParams:
    c = HcParams()
    for name in ("temperature", "d_gr", "sigma_gr", "sigma_li", "sigma_cc", "sigma_pl",
                 "d_el", "kappa_el", "t_plus", "dlnf_dlnc", "i00_grel", "i00_ceel",
                 "i00_plel", "c_gr_max", "n_const_thickness", "c_li_metal"):
        setattr(c, name, float(getattr(p, name)))
    c.faraday = float(p.constants.F)
    c.gas_constant = float(p.constants.R)
    tab = np.asarray(p.ocp_table, dtype=np.float64)
    c.n_ocp = tab.shape[0]
    for k in range(tab.shape[0]):
        c.ocp_soc[k] = tab[k, 0]
        c.ocp_v[k] = tab[k, 1]
    return c
