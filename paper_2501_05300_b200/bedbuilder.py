"""Paper bed builder: layered emission, trimming, reduced-friction relaxation and density audit
(PAPER §3.1 P:155-163 and §2.1; SPEC bed-builder S:206-278).  Host-side
orchestration; every step of the simulation runs in libdem.so.

Procedure: particles are emitted into the container from above under gravity with
friction and rolling resistance reduced to mu_t = 0.1, mu_r = 0.01 (zero at the walls) and left
to settle; a refined bed is built layer by layer from the bottom up (coarsest first), each layer
n filled to its target top, then "any excessive particles are removed" (centres above the top)
before the next layer; diameters are uniform in [0.9 d_n, 1.1 d_n].  Afterwards the full
friction (mu_t = 0.3, mu_r = 0.02) is restored.
Readings (SPEC design decisions): the emitter drops one jittered square grid plane
of spacing 1.5 d_n (staggered by half a spacing on odd planes) at a time from one diameter above
the current surface with a small downward
speed, and waits for it to come nearly to rest before the next; settled = mean kinetic energy per
particle (translational) < 1e-8 J and max |v| < 1 mm/s (budget per layer); the surface height is the mean over
2 d_max columns of the highest particle top (protocol.surface_datum).
Layer schedule: layer n (n = 0 at the surface) has diameter d_n = r^n d_min (capped at
d_max) and thickness eta d_n, its bottom at depth z_n = eta d_0 (r^{n+1} - 1)/(r - 1).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import dem as D
from .protocol import surface_datum

PAPER_MATERIAL = dict(density=2200.0, youngs=1e9, poisson=0.15, mu_t=0.3, mu_r=0.02, restitution=0.5)


class BuildTimeout(RuntimeError):
    """A layer did not settle within its budget; carries the residual KE."""

    def __init__(self, msg, ke):
        super().__init__(msg)
        self.ke = ke


def layer_schedule(d_min, d_max, r, eta, height):
    """list of (d_n, depth_top, depth_bottom), n = 0 at the surface, until `height` is
    covered; d_n = min(r^n d_min, d_max); a uniform bed is r = 1 (one layer, the full height)."""
    if not (d_min > 0 and d_max >= d_min and r >= 1 and eta >= 1 and height >= 0):
        raise ValueError("need d_max >= d_min > 0, r >= 1, eta >= 1, height >= 0")
    if height == 0:
        return []
    if r == 1.0 or d_max == d_min:
        return [(d_min, 0.0, height)]
    out, z, n = [], 0.0, 0
    while z < height - 1e-12:
        d = min(d_min * r ** n, d_max)
        if d >= d_max:                                   # the rest of the bed at d_max
            out.append((d_max, z, height))
            break
        zb = min(z + eta * d, height)
        out.append((d, z, zb))
        z, n = zb, n + 1
    return out


@dataclass
class BedSpec:
    dims: tuple                                  # container (Lx, Ly, Lz) [m]
    d_min: float
    d_max: float = None                          # None: uniform bed of d_min
    r: float = 1.0                               # layer ratio
    eta: float = 1.0                             # layer thickness in diameters
    jitter: float = 0.10                         # diameters uniform in [(1-j) d_n, (1+j) d_n]
    relax_mu: tuple = (0.1, 0.01)                # mu_t, mu_r while emitting and relaxing
    material: dict = field(default_factory=lambda: dict(PAPER_MATERIAL))
    seed: int = 0
    dt: float = None                             # None: Eq. 9 with eps 0.02 and sigma = rho g H
    n_iter_emit: int = None                      # sweeps per step while planes are emitted; None: n_iter
                                                 # (30 was measured slower: the planes take longer to calm)
    n_iter: int = None                           # sweeps per step of the settles; None: Eq. 8 (eps 0.02) on the bed's
                                                 # contact-network length n_d = sum of thickness / d_n,
                                                 # at least 30
    spacing: float = 1.5                         # emitter grid spacing / d_n
    drop_speed: float = 0.05                     # initial downward speed of emitted particles [m/s]
    ke_threshold: float = 1e-8                   # settle: mean KE per particle [J]
    v_threshold: float = 1e-3                    # settle: max |v| [m/s]
    v_emit: float = 0.02                         # next plane once max |v| is below this [m/s]
    layer_budget: float = 10.0                   # simulated seconds per layer settle (5 s; 10 here)
    plane_budget: float = 2.0                    # simulated seconds an emitted plane may take to calm down
    check_every: int = 20                        # steps between settle checks


def _emit_plane(spec, rng, d_n, z, x_lo, x_hi, gid0, stagger=0):
    """One emitter plane: a square grid of spacing spec.spacing d_n, shifted by half a spacing on
    odd planes (`stagger`) so that a plane falls into the hollows of the one below instead of
    stacking into columns, jittered within the free space between sites."""
    s = spec.spacing * d_n
    amp = 0.5 * (s - (1 + spec.jitter) * d_n) * 0.9          # jitter that keeps neighbours apart
    m = 0.5 * (1 + spec.jitter) * d_n + amp + 0.02 * d_n      # ... and clear of the walls
    off = 0.5 * s * (stagger & 1)
    xs = np.arange(x_lo[0] + m + off, x_hi[0] - m + 1e-12, s)
    ys = np.arange(x_lo[1] + m + off, x_hi[1] - m + 1e-12, s)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    n = X.size
    p = np.stack([X.ravel() + rng.uniform(-amp, amp, n), Y.ravel() + rng.uniform(-amp, amp, n),
                  np.full(n, z) + rng.uniform(0.0, 0.1 * d_n, n)], axis=1)
    rad = 0.5 * d_n * rng.uniform(1 - spec.jitter, 1 + spec.jitter, n)
    v = np.zeros((n, 3))
    v[:, 2] = -spec.drop_speed
    return p, rad, v, np.arange(gid0, gid0 + n, dtype=np.uint32)


class _World:
    """Particle arrays + their contact history; a dem.Bed is (re)created whenever the particle set
    changes (the library's bed has a fixed particle set, include/dem.h dem_set_state)."""

    def __init__(self, spec, dt, device, bed_factory=None):
        self.spec, self.dt, self.device = spec, dt, device
        self.factory = bed_factory or (lambda **kw: D.Bed(device=device, **kw))
        self.stepped = False
        self.x = np.zeros((0, 3)); self.r = np.zeros(0); self.v = np.zeros((0, 3)); self.w = np.zeros((0, 3))
        self.gid = np.zeros(0, dtype=np.uint32)
        self.layer = np.zeros(0, dtype=np.int32)
        self.hist = None
        self.bed = None
        self.t = 0.0

    def _mat(self, mu):
        m = dict(self.spec.material)
        m["mu_t"], m["mu_r"] = mu
        return m

    def open(self, mu, n_iter=None):
        self.close()
        self.n_iter_now = n_iter or self.spec.n_iter
        Lx, Ly, Lz = self.spec.dims
        self.bed = self.factory(pos=self.x, radius=self.r, vel=self.v, angvel=self.w, gid=self.gid,
                                solver=dict(dt=self.dt, n_iter=self.n_iter_now),
                                box=dict(lo=(0.0, 0.0, 0.0), hi=(Lx, Ly, Lz), wall_mask=0x3F, wall_mu_t=0.0,
                                         wall_mu_r=0.0),
                                material=self._mat(mu))
        self.stepped = False
        if self.hist is not None and len(self.x):
            self.bed.set_state(self.x, self.r, self.v, self.w, self.gid, hist=self.hist)

    def pull(self):
        if not self.stepped:             # nothing moved since the arrays were loaded
            return
        st = self.bed.get_state()
        o = np.argsort(self.gid)
        inv = np.empty_like(o)
        inv[o] = np.arange(len(o))
        # get_state is in ascending gid order; the world keeps its own order
        self.x, self.v, self.w = st["pos"][inv], st["vel"][inv], st["angvel"][inv]
        self.hist = self.bed.get_contacts() if len(self.x) else None

    def close(self):
        if self.bed is not None:
            self.bed.close()
            self.bed = None

    def add(self, p, rad, v, gid, layer):
        self.x = np.concatenate([self.x, p]); self.r = np.concatenate([self.r, rad])
        self.v = np.concatenate([self.v, v]); self.w = np.concatenate([self.w, np.zeros_like(v)])
        self.gid = np.concatenate([self.gid, gid]); self.layer = np.concatenate([self.layer, np.full(len(rad), layer)])

    def keep(self, m):
        self.x, self.r, self.v, self.w = self.x[m], self.r[m], self.v[m], self.w[m]
        self.gid, self.layer = self.gid[m], self.layer[m]

    def ke_translational(self):
        st = self.bed.get_state()
        m = self.spec.material["density"] * 4.0 / 3.0 * np.pi * st["radius"] ** 3
        return float(0.5 * (m * (st["vel"] ** 2).sum(axis=1)).sum()) / max(len(m), 1)

    def sweeps(self, n_iter):
        if self.bed is not None and n_iter and n_iter != self.n_iter_now:
            self.bed.set_solver(n_iter=n_iter)
            self.n_iter_now = n_iter

    def run_until(self, v_max, ke_max, budget, ke_any=None, strict=True):
        """Steps until max |v| < v_max and the mean translational kinetic energy per particle
        < ke_max (checked every check_every steps; the spins' share is left out: with the large
        Eq. 9 step the unconverged torques keep a small rotational jitter that carries no
        motion); returns the last report.  BuildTimeout after `budget` seconds."""
        t0 = self.t
        while True:
            rep = self.bed.step(self.spec.check_every)
            self.stepped = True
            self.t += self.spec.check_every * self.dt
            ke = rep["ke"] / max(len(self.r), 1)
            if ke_any is not None and ke < ke_any:
                return rep
            if rep["max_v"] < v_max:
                if ke < ke_max or (np.isfinite(ke_max) and self.ke_translational() < ke_max):
                    return rep
            if self.t - t0 > budget:
                if not strict:               # emission pacing: carry on with the next plane
                    return rep
                raise BuildTimeout(f"not settled after {budget} s: max |v| {rep['max_v']:.3g} m/s, "
                                   f"KE/particle {ke:.3g} J", ke)


def build_bed(spec: BedSpec, device=0, bed_factory=None):
    """Builds the bed; returns dict(pos, radius, vel, angvel, gid, layer, hist, schedule, t_sim).
    bed_factory(pos, radius, vel, angvel, gid, solver, box, material) -> bed (default: dem.Bed
    on `device`)."""
    Lx, Ly, Lz = spec.dims
    d_max = spec.d_max if spec.d_max is not None else spec.d_min
    sched = layer_schedule(spec.d_min, d_max, spec.r if spec.d_max else 1.0, spec.eta, Lz)
    rng = np.random.default_rng(spec.seed)
    rho = spec.material["density"]
    dt = spec.dt or D.plan_timestep(spec.d_min, 0.02, rho, rho * 9.81 * max(Lz, 1e-3))
    if spec.n_iter is None:
        n_d = sum((bot - top) / d for (d, top, bot) in sched) if sched else 1.0
        spec = BedSpec(**{**spec.__dict__, "n_iter": max(30, D.plan_iterations(n_d, 0.02))})
    W = _World(spec, dt, device, bed_factory)
    gid0 = 0
    try:
        for li, (d_n, dep_top, dep_bot) in enumerate(reversed(sched)):     # bottom (coarsest) layer first
            top = Lz - dep_top
            t_layer = W.t
            n_planes = 0
            while True:
                if W.bed is not None:
                    W.pull()                    # the settled positions, before measuring the surface
                surf = surface_datum(W.x, W.r, (0.5 * Lx, 0.5 * Ly), (0.5 * Lx, 0.5 * Ly), cell=2 * d_max) \
                    if len(W.r) else 0.0
                if surf >= top or surf + 1.05 * d_n > Lz:
                    break
                p, rad, v, g = _emit_plane(spec, rng, d_n, surf + 0.6 * (1 + spec.jitter) * d_n + 0.5 * d_n,
                                           (0.0, 0.0), (Lx, Ly), gid0, stagger=n_planes)
                n_planes += 1
                p[:, 2] = np.minimum(p[:, 2], Lz - 0.6 * d_n)
                gid0 += len(rad)
                W.add(p, rad, v, g, li)
                if W.bed is not None and hasattr(W.bed, "add_particles"):
                    W.bed.add_particles(p, rad, v, None, g)      # dem_add_particles: state and history kept
                    W.sweeps(spec.n_iter_emit or spec.n_iter)
                    W.stepped = False
                else:
                    W.open(spec.relax_mu, spec.n_iter_emit)
                # next plane once the bed is nearly at rest: max |v| < v_emit, or the mean kinetic
                # energy that of every sphere moving at v_emit / 4 (a single rattler may not hold it up)
                m_n = rho * np.pi / 6.0 * d_n ** 3
                # (a plane that cannot calm down within plane_budget -- spheres sliding on the
                # frictionless floor -- is buried by the next one: only the layer settle is strict)
                W.run_until(spec.v_emit, np.inf, spec.plane_budget, ke_any=0.5 * m_n * (0.25 * spec.v_emit) ** 2,
                            strict=False)
            # the layer is full: settle (Eq. 8 sweeps), then remove the excess above its top
            if W.bed is not None:
                W.sweeps(spec.n_iter)
                W.run_until(spec.v_threshold, spec.ke_threshold, spec.layer_budget)
                W.pull()
                W.keep(W.x[:, 2] <= top)
                if hasattr(W.bed, "remove_particles"):
                    W.bed.remove_particles(2, -np.inf, top)         # dem_remove_particles
                    W.stepped = False
                else:
                    W.open(spec.relax_mu)
        if W.bed is not None:
            W.run_until(spec.v_threshold, spec.ke_threshold, spec.layer_budget)
            W.pull()
            # full friction restored; the bed settles under it
            W.open((spec.material["mu_t"], spec.material["mu_r"]))
            W.run_until(spec.v_threshold, spec.ke_threshold, spec.layer_budget)
            W.pull()
    finally:
        W.close()
    o = np.argsort(W.gid)
    return dict(pos=W.x[o], radius=W.r[o], vel=W.v[o], angvel=W.w[o], gid=W.gid[o], layer=W.layer[o],
                hist=W.hist, schedule=sched, t_sim=W.t, dt=dt)


def _sphere_quadrature(n=12):
    """Equal-weight points filling the unit ball (midpoints of an n^3 grid inside it), symmetric
    under reflections, so a sphere cut by a plane through its centre splits exactly in half."""
    g = (np.arange(n) + 0.5) / n * 2 - 1
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    q = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    return q[(q ** 2).sum(axis=1) <= 1.0]


def audit_bed(pos, radius, dims, cell, rho, layer=None, schedule=None):
    """SPEC audit_bed (P:162 density check): bulk density per cubic cell with each
    sphere's mass spread over the cells it intersects (fixed quadrature of the ball), mean and
    interior-cell deviations, max overlap / d (brute force, small beds), and the mixing metric:
    fraction of particles farther than one own diameter outside their layer's band."""
    pos, radius = np.asarray(pos, float), np.asarray(radius, float)
    if len(radius) and cell < 2 * radius.max():
        raise ValueError("cells must be at least d_max wide (they must hold several particles)")
    nc = [max(1, int(np.floor(dims[k] / cell + 1e-9))) for k in range(3)]
    grid = np.zeros(nc)
    q = _sphere_quadrature()
    for x, r in zip(pos, radius):
        m = rho * 4.0 / 3.0 * np.pi * r ** 3
        pts = x + r * q
        ijk = np.floor(pts / cell).astype(np.int64)
        for k in range(3):
            ijk[:, k] = np.clip(ijk[:, k], 0, nc[k] - 1)
        np.add.at(grid, (ijk[:, 0], ijk[:, 1], ijk[:, 2]), m / len(q))
    dens = grid / cell ** 3
    out = dict(density=dens, mean=float(dens.mean()))
    if min(nc) >= 3:
        inner = dens[1:-1, 1:-1, 1:-2] if nc[2] >= 4 else dens[1:-1, 1:-1, :]
        out["interior_mean"] = float(inner.mean())
        out["interior_max_dev"] = float(np.abs(inner / inner.mean() - 1).max()) if inner.mean() > 0 else 0.0
    if len(radius) > 1 and len(radius) <= 20000:
        from scipy.spatial import cKDTree
        tree = cKDTree(pos)
        pairs = tree.query_pairs(2 * radius.max(), output_type="ndarray")
        if len(pairs):
            d = np.linalg.norm(pos[pairs[:, 0]] - pos[pairs[:, 1]], axis=1)
            ov = (radius[pairs[:, 0]] + radius[pairs[:, 1]] - d) / (2 * np.minimum(radius[pairs[:, 0]], radius[pairs[:, 1]]))
            out["max_overlap_ratio"] = float(max(ov.max(), 0.0))
        else:
            out["max_overlap_ratio"] = 0.0
    if layer is not None and schedule is not None and len(radius):
        H = dims[2]
        bands = list(reversed(schedule))                    # layer index 0 = bottom band
        lo = np.array([H - b[2] for b in bands])[layer]
        hi = np.array([H - b[1] for b in bands])[layer]
        z = pos[:, 2]
        out["mixing"] = float(np.mean((z < lo - 2 * radius) | (z > hi + 2 * radius)))
    return out
