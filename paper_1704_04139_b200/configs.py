"""The BASELINE.json configurations expressed as :class:`CellSpec` + run settings."""

from __future__ import annotations

from dataclasses import dataclass

from .microgen import CellSpec


@dataclass
class RunSpec:
    name: str
    cell: CellSpec
    c_rate: float
    dt: float
    n_steps: int
    soc_init: float = 0.1
    i00_plel_exchange: float = 1e-3   # plating exchange current density at c_el_init, A/m^2


CONFIGS = {
    "tiny": RunSpec("tiny", CellSpec(32, 32, 64, 28, 8, seed=0, radius_mean=4.0, porosity=0.35),
                    c_rate=1.0, dt=1.0, n_steps=10),
    "medium": RunSpec("medium", CellSpec(64, 64, 128, 56, 16, seed=1, radius_mean=6.0, porosity=0.35),
                      c_rate=2.0, dt=0.5, n_steps=20),
    "large": RunSpec("large", CellSpec(128, 128, 256, 112, 32, seed=2, radius_mean=6.0, porosity=0.30),
                     c_rate=3.0, dt=0.25, n_steps=200),
}
