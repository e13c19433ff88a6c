"""Seeded microstructure setup for the BASELINE configurations.

The reference generates half cells with a Laguerre / Gaussian-random-field
pipeline (``src/halfcell/microgen/generate.py:87-153``).  BASELINE.json's
configurations instead specify a union of balls with Poisson centres and
Gamma-distributed radii thresholded to a target porosity; that is what
:func:`generate_cell` builds.  The slab assembly (working collector at z = 0,
a pore layer capping the electrode, pruning of graphite not connected to the
collector) and the germ-grain plated-lithium layer follow the reference
(``generate.py:71-84,131-135`` and ``plating.py:53-109``), so every grid is
a valid reference ``PhaseGrid`` and can be fed to both the reference operator
and this package.

Geometry setup runs once per cell and is not on the timed path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy import ndimage

from .errors import GeometryError
from .phases import Phase, PhaseGrid

_FACE_OFFSETS = np.array([(0, 0, 1), (0, 0, -1), (0, 1, 0), (0, -1, 0), (1, 0, 0), (-1, 0, 0)])


@dataclass
class CellSpec:
    """One BASELINE cell: grid, z-layer split and ball statistics (lengths in voxels)."""

    nx: int
    ny: int
    nz: int
    n_anode: int           # z layers [0, n_anode): working collector at z=0 + graphite electrode
    n_separator: int       # pure electrolyte
    seed: int = 0
    radius_mean: float = 4.0
    gamma_shape: float = 4.0
    porosity: float = 0.35
    voxel_size: float = 1.0            # um
    plating_intensity: float = 0.01    # germs per um^2 (reference GenConfig default)
    plating_radius: float = 2.2        # um

    @property
    def n_counter(self) -> int:
        return self.nz - self.n_anode - self.n_separator


def sample_germs(extent_x: float, extent_y: float, intensity: float,
                 rng: np.random.Generator) -> np.ndarray:
    """Poisson germs on a rectangle; same draw order as reference ``plating.py:16-23``."""
    n = rng.poisson(intensity * extent_x * extent_y)
    pts = np.empty((n, 2))
    pts[:, 0] = rng.random(n) * extent_x
    pts[:, 1] = rng.random(n) * extent_y
    return pts


def _min_d2(points: np.ndarray, stars: np.ndarray, chunk: int = 4096) -> np.ndarray:
    out = np.empty(points.shape[0])
    for s in range(0, points.shape[0], chunk):
        d = points[s:s + chunk, None, :] - stars[None, :, :]
        out[s:s + chunk] = np.min(np.sum(d ** 2, axis=2), axis=1)
    return out


def plate_germs(grid: PhaseGrid, intensity: float, grain_radius: float,
                rng: np.random.Generator) -> PhaseGrid:
    """Germ-grain plated-lithium layer (algorithm of reference ``plating.py:53-109``).

    Germs on the separator plane are projected down their column onto the top
    graphite voxel; electrolyte face-neighbours of graphite surface voxels
    that lie, with their own centre, inside a grain ball become PLATED_LI.
    """
    labels = grid.labels.copy()
    nz, ny, nx = labels.shape
    h = grid.voxel_size
    germs = sample_germs(nx * h, ny * h, intensity, rng)
    if germs.shape[0] == 0:
        return PhaseGrid(labels, h)
    gr = labels == Phase.GRAPHITE
    gr_z = np.nonzero(gr.any(axis=(1, 2)))[0]
    if gr_z.size == 0:
        return PhaseGrid(labels, h)
    z_top = int(gr_z.max())
    el = labels == Phase.ELECTROLYTE
    near_el = np.zeros_like(el)
    near_el[1:] |= el[:-1]
    near_el[:-1] |= el[1:]
    near_el[:, 1:] |= el[:, :-1]
    near_el[:, :-1] |= el[:, 1:]
    near_el[:, :, 1:] |= el[:, :, :-1]
    near_el[:, :, :-1] |= el[:, :, 1:]
    surf = np.argwhere(gr & near_el)
    if surf.size == 0:
        return PhaseGrid(labels, h)
    ix = np.minimum(nx - 1, (germs[:, 0] / h).astype(np.int64))
    iy = np.minimum(ny - 1, (germs[:, 1] / h).astype(np.int64))
    cols = gr[: z_top + 1, iy, ix]                       # (z, germ)
    has = cols.any(axis=0)
    if not has.any():
        return PhaseGrid(labels, h)
    z_hit = z_top - np.argmax(cols[::-1], axis=0)        # highest graphite voxel per column
    stars = np.stack([germs[has, 0], germs[has, 1], (z_hit[has] + 1) * h], axis=1)
    r2 = grain_radius ** 2
    surf_c = (surf[:, ::-1] + 0.5) * h
    # only surface voxels that can be within reach of a star matter
    sel = surf[_min_d2(surf_c, stars) <= r2]
    for dz, dy, dx in _FACE_OFFSETS:
        nb = sel + np.array([dz, dy, dx])
        ok = ((nb[:, 0] >= 0) & (nb[:, 0] < nz) & (nb[:, 1] >= 0) & (nb[:, 1] < ny)
              & (nb[:, 2] >= 0) & (nb[:, 2] < nx))
        nb = nb[ok]
        nb = nb[el[nb[:, 0], nb[:, 1], nb[:, 2]]]
        if nb.size == 0:
            continue
        inside = _min_d2((nb[:, ::-1] + 0.5) * h, stars) <= r2
        nb = nb[inside]
        labels[nb[:, 0], nb[:, 1], nb[:, 2]] = Phase.PLATED_LI
    return PhaseGrid(labels, h)


def prune_disconnected_graphite(labels: np.ndarray, z_contact: int) -> np.ndarray:
    """Graphite not 6-connected to the collector contact layer becomes electrolyte
    (reference ``generate.py:71-84``)."""
    gr = labels == Phase.GRAPHITE
    comp, n = ndimage.label(gr, structure=ndimage.generate_binary_structure(3, 1))
    if n == 0:
        raise GeometryError("generation produced no graphite")
    touching = np.unique(comp[z_contact][comp[z_contact] > 0])
    if touching.size == 0:
        raise GeometryError("no graphite component touches the working collector")
    out = labels.copy()
    out[gr & ~np.isin(comp, touching)] = Phase.ELECTROLYTE
    return out


def ball_union_solid(shape_zyx, radius_mean, gamma_shape, porosity, rng) -> np.ndarray:
    """Union-of-balls solid mask with exactly the target porosity.

    Centres are a Poisson process whose intensity gives the target porosity for
    the Boolean model; radii ~ Gamma(shape, mean).  The solid is the
    super-level set ``max_i (r_i - |x - c_i|) >= t`` with ``t`` the porosity
    quantile, so the voxel porosity is hit exactly.
    """
    nz, ny, nx = shape_zyx
    theta = radius_mean / gamma_shape
    er3 = theta ** 3 * gamma_shape * (gamma_shape + 1) * (gamma_shape + 2)
    m = float(radius_mean)               # centres also fall in a margin around the box
    ext = np.array([nx + 2 * m, ny + 2 * m, nz + 2 * m])
    n_mean = -np.log(porosity) * float(np.prod(ext)) / (4.0 / 3.0 * np.pi * er3)
    n = int(rng.poisson(n_mean))
    centres = rng.random((n, 3)) * ext - m
    radii = rng.gamma(gamma_shape, theta, size=n)
    f = np.full(shape_zyx, -np.inf)
    for (cx, cy, cz), r in zip(centres, radii):
        reach = r + 2.0
        x0, x1 = max(0, int(cx - reach)), min(nx, int(cx + reach) + 1)
        y0, y1 = max(0, int(cy - reach)), min(ny, int(cy + reach) + 1)
        z0, z1 = max(0, int(cz - reach)), min(nz, int(cz + reach) + 1)
        if x0 >= x1 or y0 >= y1 or z0 >= z1:
            continue
        zz = (np.arange(z0, z1) + 0.5 - cz)[:, None, None]
        yy = (np.arange(y0, y1) + 0.5 - cy)[None, :, None]
        xx = (np.arange(x0, x1) + 0.5 - cx)[None, None, :]
        val = r - np.sqrt(xx * xx + yy * yy + zz * zz)
        np.maximum(f[z0:z1, y0:y1, x0:x1], val, out=f[z0:z1, y0:y1, x0:x1])
    n_solid = int(round((1.0 - porosity) * f.size))
    if n_solid <= 0:
        return np.zeros(shape_zyx, dtype=bool)
    t = np.partition(f.ravel(), f.size - n_solid)[f.size - n_solid]
    if not np.isfinite(t):
        raise GeometryError("too few balls to reach the target solid fraction")
    return f >= t


def generate_cell(spec: CellSpec) -> PhaseGrid:
    """Assemble one half cell from a :class:`CellSpec`.

    z layout: 0 working collector | 1..n_anode-1 graphite electrode (top layer
    kept as pore) | separator electrolyte | lithium-foil counter electrode |
    counter collector at z = nz - 1 (the grounded face).
    """
    if spec.n_anode < 3 or spec.n_separator < 1 or spec.n_counter < 2:
        raise GeometryError("layer split leaves no room for collector/electrode/foil")
    ss_balls, ss_plate = np.random.SeedSequence(spec.seed).spawn(2)
    labels = np.full((spec.nz, spec.ny, spec.nx), Phase.ELECTROLYTE, dtype=np.uint8)
    labels[0] = Phase.COLLECTOR_WORKING
    e0, e1 = 1, spec.n_anode - 1          # electrode slab without its pore cap
    solid = ball_union_solid((e1 - e0, spec.ny, spec.nx), spec.radius_mean,
                             spec.gamma_shape, spec.porosity, np.random.default_rng(ss_balls))
    labels[e0:e1][solid] = Phase.GRAPHITE
    f0 = spec.n_anode + spec.n_separator
    labels[f0:spec.nz - 1] = Phase.LI_FOIL
    labels[spec.nz - 1] = Phase.COLLECTOR_COUNTER
    labels = prune_disconnected_graphite(labels, e0)
    grid = PhaseGrid(labels, spec.voxel_size)
    return plate_germs(grid, spec.plating_intensity, spec.plating_radius,
                       np.random.default_rng(ss_plate))
