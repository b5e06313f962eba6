"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no contact law, no solver, no integrator):
it only places spheres.  Recipes follow SURVEY.md §8(d) / DESIGN.md §4:

* radius jitter r = r_nom * U[0.9, 1.1] ("uniformly randomized in the range 0.9 d_n
  to 1.1 d_n");
* config 0: simple-cubic 16^3 lattice at 7 mm, +-0.3 mm jitter, r in [2.7, 3.3] mm,
  box widened to 0.1122 m in x/y (reading R25);
* configs 1-4: banded (or graded) beds on FCC / square lattices whose size grows with depth
  (Eq. 1 and the layer construction of Fig. 2), seeded per gid.

Random numbers come from numpy's Philox bit generator keyed by the seed.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Bed:
    x: np.ndarray            # (n,3) float64 positions
    r: np.ndarray            # (n,) float64 radii
    v: np.ndarray            # (n,3) float64
    w: np.ndarray            # (n,3) float64
    gid: np.ndarray          # (n,) uint32
    box_lo: tuple
    box_hi: tuple
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n(self):
        return len(self.r)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(int(seed)))


# ----------------------------------------------------------------------------- config 0

def config0(seed: int = 1000) -> Bed:
    """BASELINE.json configs[0]: 4,096 spheres, r ~ U[2.7,3.3] mm, SC lattice 7 mm, jitter
    +-0.3 mm, walled box (x/y widened to 0.1122 m, reading R25), at rest."""
    rng = _rng(seed)
    n1 = 16
    a = 7e-3
    L = 0.1122
    off = 0.5 * (L - (n1 - 1) * a)
    k, j, i = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    x = np.stack([off + i.ravel() * a, off + j.ravel() * a, 3.6e-3 + k.ravel() * a], axis=1)
    x += rng.uniform(-0.3e-3, 0.3e-3, size=x.shape)
    r = rng.uniform(2.7e-3, 3.3e-3, size=len(x))
    n = len(x)
    return Bed(x=x, r=r, v=np.zeros((n, 3)), w=np.zeros((n, 3)), gid=np.arange(n, dtype=np.uint32),
               box_lo=(0.0, 0.0, 0.0), box_hi=(L, L, 0.12), name="config0")


# ----------------------------------------------------------------------------- lattice helpers

def _fcc_sites(lo, hi, a):
    """FCC sites (nearest-neighbour distance a) inside the box [lo, hi], plane-major from the
    bottom, then y, then x."""
    A = a * np.sqrt(2.0)
    basis = np.array([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]]) * A
    n = [int(np.floor((hi[d] - lo[d]) / A)) + 2 for d in range(3)]
    out = []
    # build by half-cell planes so that the order is plane-major
    for kz in range(2 * n[2]):
        z = lo[2] + 0.5 * A * kz
        if z > hi[2] + 1e-12:
            break
        sub = basis[np.isclose(basis[:, 2], 0.5 * A * (kz % 2))]
        ii, jj = np.meshgrid(np.arange(n[0]), np.arange(n[1]), indexing="xy")
        for b in sub:
            xs = lo[0] + b[0] + ii.ravel() * A
            ys = lo[1] + b[1] + jj.ravel() * A
            pts = np.stack([xs, ys, np.full_like(xs, z)], axis=1)
            m = (pts[:, 0] <= hi[0] + 1e-12) & (pts[:, 1] <= hi[1] + 1e-12)
            out.append(pts[m])
    if not out:
        return np.zeros((0, 3))
    pts = np.concatenate(out)
    order = np.lexsort((pts[:, 0], pts[:, 1], pts[:, 2]))
    return pts[order]


def _square_plane(lo, hi, z, s):
    nx = int(np.floor((hi[0] - lo[0]) / s)) + 1
    ny = int(np.floor((hi[1] - lo[1]) / s)) + 1
    ii, jj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    xs = lo[0] + ii.ravel() * s
    ys = lo[1] + jj.ravel() * s
    return np.stack([xs, ys, np.full_like(xs, z)], axis=1)


def banded_bed(dims, bands, seed, spacing=2.25, jitter=0.01, name="banded") -> Bed:
    """Bed in the box [0,dims]; bands = [(depth_top, depth_bottom, r_nom), ...] with depth
    measured down from the top z = dims[2] (P:67 uses depth).  Each band is an FCC lattice
    with nearest-neighbour distance spacing*r_nom kept 1.1 r_nom away from the band faces and
    the walls, so no two spheres overlap at t=0."""
    rng = _rng(seed)
    H = dims[2]
    xs, rs = [], []
    for (d_top, d_bot, rn) in sorted(bands, key=lambda b: -b[1]):   # bottom band first
        m = 1.1 * rn
        lo = (m, m, H - d_bot + m)
        hi = (dims[0] - m, dims[1] - m, H - d_top - m)
        if hi[2] < lo[2]:
            continue
        p = _fcc_sites(lo, hi, spacing * rn)
        xs.append(p)
        rs.append(np.full(len(p), rn))
    x = np.concatenate(xs)
    rn = np.concatenate(rs)
    x = x + rng.uniform(-jitter, jitter, size=x.shape) * rn[:, None]
    r = rn * rng.uniform(0.9, 1.1, size=len(rn))
    n = len(r)
    return Bed(x=x, r=r, v=np.zeros((n, 3)), w=np.zeros((n, 3)), gid=np.arange(n, dtype=np.uint32),
               box_lo=(0.0, 0.0, 0.0), box_hi=tuple(dims), name=name, meta={"bands": bands})


def graded_bed(dims, r_top, r_bot, depth_grad, seed, spacing=2.25, jitter=0.01, name="graded") -> Bed:
    """Radius growing linearly with depth from r_top at the surface to r_bot at depth_grad
    (Eq. 1 with d = 2r), square-lattice planes with in-plane spacing spacing*r_k and vertical
    gap 0.5*spacing*(r_k + r_{k+1}), built from the bottom up."""
    rng = _rng(seed)
    H = dims[2]

    def rnom(z):
        depth = H - z
        return r_top + (r_bot - r_top) * min(max(depth / depth_grad, 0.0), 1.0)

    planes, radii = [], []
    z = 1.1 * rnom(0.0)
    while True:
        rk = rnom(z)
        if z + 1.1 * rk > H:
            break
        m = 1.1 * rk
        p = _square_plane((m, m), (dims[0] - m, dims[1] - m), z, spacing * rk)
        planes.append(p)
        radii.append(np.full(len(p), rk))
        zn = z + spacing * rk
        for _ in range(4):
            zn = z + 0.5 * spacing * (rk + rnom(zn))
        z = zn
    x = np.concatenate(planes)
    rn = np.concatenate(radii)
    x = x + rng.uniform(-jitter, jitter, size=x.shape) * rn[:, None]
    r = rn * rng.uniform(0.9, 1.1, size=len(rn))
    n = len(r)
    return Bed(x=x, r=r, v=np.zeros((n, 3)), w=np.zeros((n, 3)), gid=np.arange(n, dtype=np.uint32),
               box_lo=(0.0, 0.0, 0.0), box_hi=tuple(dims), name=name)


def config_bed(cfg: int, variant: str = "geom", seed: int | None = None, x_scale: float = 1.0) -> Bed:
    """BASELINE.json configs 1-4.  variant 'count' lengthens x to reach
    the stated count (reading R27); x_scale shrinks x for mini beds."""
    seed = 1000 + cfg if seed is None else seed
    if cfg == 0:
        return config0(seed)
    if cfg == 1:
        dims = (0.4 * x_scale, 0.4, 0.3)
        return banded_bed(dims, [(0.0, 0.06, 2e-3), (0.06, 0.3, 4e-3)], seed, name="config1")
    if cfg == 2:
        L = (7.8 if variant == "count" else 1.0) * x_scale
        return graded_bed((L, 0.5, 0.5), 2e-3, 16e-3, 0.5, seed, name=f"config2-{variant}")
    if cfg == 3:
        L = (4.3 if variant == "count" else 1.0) * x_scale
        return banded_bed((L, 0.5, 0.3), [(0.0, 0.3, 2e-3)], seed, name=f"config3-{variant}")
    if cfg == 4:
        L = (29.6 if variant == "count" else 8.0) * x_scale
        return banded_bed((L, 1.0, 0.6), [(0.0, 0.08, 2e-3), (0.08, 0.25, 6e-3), (0.25, 0.6, 16e-3)],
                          seed, name=f"config4-{variant}")
    raise ValueError(cfg)


# ----------------------------------------------------------------------------- random clouds

def random_cloud(n, box_lo, box_hi, r_min, r_max, seed, v_scale=0.0, w_scale=0.0, loguniform=False) -> Bed:
    """n spheres uniformly in a box with radii in [r_min, r_max] (log-uniform for strongly
    polydisperse clouds), random velocities/spins.  Overlaps are allowed (parity edge cases)."""
    rng = _rng(seed)
    lo, hi = np.asarray(box_lo, float), np.asarray(box_hi, float)
    x = lo + (hi - lo) * rng.random((n, 3))
    if loguniform:
        r = np.exp(rng.uniform(np.log(r_min), np.log(r_max), size=n))
    else:
        r = rng.uniform(r_min, r_max, size=n)
    v = rng.normal(0.0, 1.0, size=(n, 3)) * v_scale
    w = rng.normal(0.0, 1.0, size=(n, 3)) * w_scale
    gid = rng.permutation(n).astype(np.uint32)
    return Bed(x=x, r=r, v=v, w=w, gid=gid, box_lo=tuple(lo), box_hi=tuple(hi), name="cloud")


# ----------------------------------------------------------------------------- x-slab pieces

def shift_slab(bed: Bed, rank: int, world: int) -> tuple:
    """Rank r's piece of a bed made of `world` copies of `bed`'s box laid end to end along x
    (each copy generated with its own seed by the caller): positions shifted by r L, gids offset
    by r n (unique over the job), box spanning all pieces.  Returns (bed, (slab_lo, slab_hi))."""
    L = bed.box_hi[0] - bed.box_lo[0]
    x = bed.x.copy()
    x[:, 0] += rank * L
    gid = (bed.gid.astype(np.int64) + rank * bed.n).astype(np.uint32)
    lo = bed.box_lo[0] + rank * L
    out = Bed(x=x, r=bed.r, v=bed.v, w=bed.w, gid=gid, box_lo=bed.box_lo,
              box_hi=(bed.box_lo[0] + world * L,) + tuple(bed.box_hi[1:]), name=f"{bed.name}-slab{rank}of{world}",
              meta=dict(bed.meta))
    return out, (lo, lo + L)
