"""Thin ctypes binding of libdem.so (include/dem.h): argument marshalling only.

Every step of the DEM path runs in the library's CUDA kernels; there is no Python or CPU
fallback.  If ``lib/libdem.so`` is missing the import fails loudly.  PyTorch is used for
plumbing only: the CUDA stream the library issues on and (optionally) its caching allocator.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DEM_LIB_VARIANT") or os.path.join(HERE, "lib", "libdem.so")

DEM_OK, DEM_ERR_INVALID, DEM_ERR_DIVERGED, DEM_ERR_STATE, DEM_ERR_CUDA, DEM_ERR_NCCL, DEM_ERR_OOM = 0, 2, 3, 4, 5, 6, 7
AXIS_LOCKED, AXIS_VELOCITY, AXIS_FORCE = 0, 1, 2
WALL_KEY_BASE = 0xFFFFFFF0
PLATE_KEY_BASE = 0xFFFFF000


class DemError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"dem status {status}: {msg}")
        self.status = status


class DivergedError(DemError):
    pass


class Material(C.Structure):
    _fields_ = [("density", C.c_double), ("youngs", C.c_double), ("poisson", C.c_double),
                ("mu_t", C.c_double), ("mu_r", C.c_double), ("restitution", C.c_double)]


class Solver(C.Structure):
    _fields_ = [("dt", C.c_double), ("n_iter", C.c_int32), ("n_iter_impact", C.c_int32),
                ("hertz_exp", C.c_double), ("k_lin", C.c_double), ("damping_steps", C.c_double),
                ("v_impact", C.c_double), ("gravity", C.c_double * 3), ("rolling_dims", C.c_int32),
                ("ordering", C.c_int32), ("skin", C.c_double), ("reduction", C.c_int32), ("plate_coupling", C.c_int32)]


class Box(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("wall_mask", C.c_uint32), ("pad0", C.c_uint32),
                ("wall_mu_t", C.c_double), ("wall_mu_r", C.c_double)]


class Particles(C.Structure):
    _fields_ = [("n", C.c_int64), ("pos", C.c_void_p), ("radius", C.c_void_p), ("vel", C.c_void_p),
                ("angvel", C.c_void_p), ("gid", C.c_void_p), ("on_device", C.c_int32), ("pad0", C.c_int32)]


class Generator(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_bands", C.c_int32), ("band_bottom_depth", C.c_void_p),
                ("band_r_nom", C.c_void_p), ("d_min", C.c_double), ("gamma", C.c_double), ("d_max", C.c_double),
                ("ratio_r", C.c_double), ("eta", C.c_double), ("spacing_factor", C.c_double),
                ("pos_jitter", C.c_double), ("size_jitter", C.c_double), ("seed", C.c_uint64)]


class BedDesc(C.Structure):
    _fields_ = [("struct_size", C.c_size_t), ("mat", Material), ("solver", Solver), ("box", Box),
                ("parts", Particles), ("source", C.c_int32), ("pad0", C.c_int32), ("gen", Generator)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class DistDesc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world_size", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("cuda_stream", C.c_void_p), ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", C.c_void_p),
                ("slab_lo", C.c_double), ("slab_hi", C.c_double), ("transport", C.c_int32), ("pad0", C.c_int32),
                ("loopback", C.c_void_p)]


class StepReport(C.Structure):
    _fields_ = [("step", C.c_int64), ("time", C.c_double), ("n_contacts", C.c_int64), ("n_pp", C.c_int64),
                ("n_wall", C.c_int64), ("n_plate", C.c_int64), ("n_degenerate", C.c_int64),
                ("n_candidates", C.c_int64), ("impact_fired", C.c_int32), ("rebuilt", C.c_int32),
                ("ke", C.c_double), ("max_v", C.c_double), ("max_disp", C.c_double),
                ("n_iter", C.c_int32), ("n_iter_impact", C.c_int32), ("n_colors", C.c_int32), ("pad0", C.c_int32),
                ("max_normal_residual", C.c_double), ("max_cone_excess", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class StateView(C.Structure):
    _fields_ = [("n", C.c_int64), ("pos", C.c_void_p), ("vel", C.c_void_p), ("angvel", C.c_void_p),
                ("radius", C.c_void_p), ("gid", C.c_void_p), ("on_device", C.c_int32), ("pad0", C.c_int32)]


class ContactView(C.Structure):
    _fields_ = [("n", C.c_int64), ("key", C.c_void_p), ("normal", C.c_void_p), ("delta", C.c_void_p),
                ("P", C.c_void_p), ("on_device", C.c_int32), ("pad0", C.c_int32)]


class PlateDesc(C.Structure):
    _fields_ = [("n_boxes", C.c_int32), ("pad0", C.c_int32), ("lo", C.c_void_p), ("hi", C.c_void_p),
                ("mass", C.c_double), ("mu_t", C.c_double), ("mu_r", C.c_double)]


class PlateState(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("vel", C.c_double * 3), ("force", C.c_double * 3),
                ("motor_force", C.c_double * 3), ("n_contacts", C.c_int64)]


class WallState(C.Structure):
    _fields_ = [("point", C.c_double * 3), ("normal", C.c_double * 3), ("velocity", C.c_double),
                ("force", C.c_double * 3), ("n_contacts", C.c_int64)]


class Timing(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_detect", C.c_double), ("ms_rebuild", C.c_double),
                ("ms_sweeps", C.c_double), ("ms_integrate", C.c_double), ("n_sweep_launches", C.c_int64),
                ("n_kernel_launches", C.c_int64), ("contact_sweeps", C.c_int64), ("particle_sweeps", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


CONTACT_DTYPE = np.dtype([("key", "<u8"), ("n", "<f8", (3,)), ("delta", "<f8"), ("P", "<f8", (7,))])

# every symbol include/dem.h declares (checked by tests/test_boundary.py)
EXPORTS = ["dem_create_bed", "dem_step", "dem_set_solver", "dem_get_state", "dem_set_state", "dem_get_contacts", "dem_get_forces",
           "dem_add_plate", "dem_drive_plate", "dem_get_plate", "dem_drive_wall", "dem_get_wall", "dem_set_timing",
           "dem_get_timing", "dem_rebalance", "dem_add_particles", "dem_remove_particles",
           "dem_reset_timing", "dem_bench_sweeps", "dem_drive_upload_bytes", "dem_num_particles", "dem_num_local", "dem_nccl_unique_id",
           "dem_loopback_create", "dem_loopback_destroy", "dem_generator_count", "dem_stream", "dem_destroy", "dem_last_error", "dem_profile_diameter",
           "dem_contact_network_length", "dem_plan_iterations", "dem_plan_timestep"]

_lib = None


def lib():
    """Load libdem.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.dem_create_bed.argtypes = [C.POINTER(BedDesc), C.POINTER(DistDesc), C.POINTER(vp)]
        L.dem_step.argtypes = [vp, i32, C.POINTER(StepReport)]
        L.dem_set_solver.argtypes = [vp, C.POINTER(Solver)]
        L.dem_get_state.argtypes = [vp, C.POINTER(StateView)]
        L.dem_set_state.argtypes = [vp, C.POINTER(StateView), C.POINTER(ContactView)]
        L.dem_get_contacts.argtypes = [vp, C.POINTER(ContactView)]
        L.dem_get_forces.argtypes = [vp, vp, vp, i32]
        L.dem_add_plate.argtypes = [vp, C.POINTER(PlateDesc), C.POINTER(C.c_double), C.POINTER(i32)]
        L.dem_drive_plate.argtypes = [vp, i32, i32, i32, d, d, d, d]
        L.dem_get_plate.argtypes = [vp, i32, C.POINTER(PlateState)]
        L.dem_drive_wall.argtypes = [vp, i32, d]
        L.dem_get_wall.argtypes = [vp, i32, C.POINTER(WallState)]
        L.dem_rebalance.argtypes = [vp, i32, C.POINTER(C.c_double)]
        L.dem_add_particles.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, i32]
        L.dem_add_particles.restype = C.c_int
        L.dem_remove_particles.argtypes = [vp, i32, d, d, C.POINTER(C.c_int64)]
        L.dem_remove_particles.restype = C.c_int
        L.dem_rebalance.restype = C.c_int
        L.dem_set_timing.argtypes = [vp, i32]
        L.dem_get_timing.argtypes = [vp, C.POINTER(Timing)]
        L.dem_reset_timing.argtypes = [vp]
        L.dem_bench_sweeps.argtypes = [vp, i32, i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        if hasattr(L, "dem_drive_upload_bytes"):      # (diagnostic builds of older libraries lack it)
            L.dem_drive_upload_bytes.argtypes = []
            L.dem_drive_upload_bytes.restype = C.c_int64
        L.dem_num_particles.argtypes = [vp]
        L.dem_num_particles.restype = C.c_int64
        L.dem_num_local.argtypes = [vp]
        L.dem_num_local.restype = C.c_int64
        L.dem_nccl_unique_id.argtypes = [vp]
        L.dem_nccl_unique_id.restype = C.c_int
        L.dem_loopback_create.argtypes = [i32]
        L.dem_loopback_create.restype = vp
        L.dem_loopback_destroy.argtypes = [vp]
        L.dem_loopback_destroy.restype = None
        L.dem_generator_count.argtypes = [C.POINTER(Generator), C.POINTER(Box), d, d, C.POINTER(C.c_int64)]
        L.dem_generator_count.restype = C.c_int
        L.dem_stream.argtypes = [vp]
        L.dem_stream.restype = vp
        L.dem_destroy.argtypes = [vp]
        L.dem_last_error.argtypes = [vp]
        L.dem_last_error.restype = C.c_char_p
        L.dem_profile_diameter.argtypes = [d, d, d, d]
        L.dem_profile_diameter.restype = d
        L.dem_contact_network_length.argtypes = [d, d, d, d, d]
        L.dem_contact_network_length.restype = d
        L.dem_plan_iterations.argtypes = [d, d]
        L.dem_plan_iterations.restype = i32
        L.dem_plan_timestep.argtypes = [d, d, d, d]
        L.dem_plan_timestep.restype = d
        for f in ["dem_create_bed", "dem_step", "dem_set_solver", "dem_get_state", "dem_set_state", "dem_get_contacts",
                  "dem_get_forces", "dem_add_plate", "dem_drive_plate", "dem_get_plate", "dem_drive_wall",
                  "dem_get_wall", "dem_set_timing", "dem_get_timing", "dem_reset_timing", "dem_bench_sweeps", "dem_destroy"]:
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


# ---------------------------------------------------------------- planner helpers (host-only)
def profile_diameter(d_min, d_max, gamma, depth):
    return lib().dem_profile_diameter(d_min, d_max, gamma, depth)


def contact_network_length(d_min, d_max, r, eta, h):
    return lib().dem_contact_network_length(d_min, d_max, r, eta, h)


def plan_iterations(n_d, eps=0.02):
    return lib().dem_plan_iterations(n_d, eps)


def plan_timestep(d, eps, rho, sigma):
    return lib().dem_plan_timestep(d, eps, rho, sigma)


# ---------------------------------------------------------------- x-slab decomposition plumbing
def boundary_upload_bytes():
    """bytes one dem_drive_wall / dem_drive_plate call copies host -> device (dem_drive_upload_bytes)"""
    return int(lib().dem_drive_upload_bytes())


def nccl_unique_id():
    """A fresh ncclUniqueId (128 bytes) for rank 0 to broadcast (torch.distributed)."""
    buf = (C.c_ubyte * 128)()
    st = lib().dem_nccl_unique_id(buf)
    if st != DEM_OK:
        raise DemError(st, lib().dem_last_error(None).decode())
    return bytes(buf)


class LoopbackGroup:
    """world_size ranks inside one process (one host thread per rank) exchanging ghosts with
    device copies: the decomposition on a single GPU (include/dem.h)."""

    def __init__(self, world_size):
        import weakref
        self.world_size = world_size
        self.handle = lib().dem_loopback_create(world_size)
        self._beds = weakref.WeakSet()

    def close(self):
        """Destroys the group; beds still open on it are closed first (their transports point
        into the group)."""
        if self.handle:
            for b in list(self._beds):
                b.close()
            lib().dem_loopback_destroy(self.handle)
            self.handle = None


def slab_bounds(x, world_size, lo, hi):
    """Slab faces at particle-count quantiles of x; outer faces at the box."""
    import numpy as _np
    q = _np.quantile(_np.asarray(x, float), _np.arange(1, world_size) / world_size) if world_size > 1 else []
    return [lo] + [float(v) for v in q] + [hi]


# ---------------------------------------------------------------- on-device generator (include/dem.h)
def make_generator(kind="bands", bands=(), d_min=0.0, gamma=0.0, d_max=0.0, ratio_r=0.0, eta=0.0,
                   spacing_factor=2.25, pos_jitter=0.01, size_jitter=0.10, seed=0):
    """dem_generator: kind 'bands' with bands = [(depth_bottom, r_nom), ...] (top band first),
    'profile' (Eq. 1: d_min, gamma, d_max) or 'layers' (Fig. 2: d_min, d_max, ratio_r, eta).
    Returns (Generator, keep-alive arrays)."""
    g = Generator()
    g.kind = {"bands": 0, "profile": 1, "layers": 2}[kind]
    keep = ()
    if g.kind == 0:
        bd = np.ascontiguousarray([b[0] for b in bands], dtype=np.float64)
        br = np.ascontiguousarray([b[1] for b in bands], dtype=np.float64)
        g.n_bands, g.band_bottom_depth, g.band_r_nom = len(bd), bd.ctypes.data, br.ctypes.data
        keep = (bd, br)
    g.d_min, g.gamma, g.d_max, g.ratio_r, g.eta = d_min, gamma, d_max, ratio_r, eta
    g.spacing_factor, g.pos_jitter, g.size_jitter, g.seed = spacing_factor, pos_jitter, size_jitter, seed
    return g, keep


def _box(box):
    bx = dict(lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0), wall_mask=0x3F, wall_mu_t=0.0, wall_mu_r=0.0)
    bx.update(box or {})
    b = Box()
    for j in range(3):
        b.lo[j], b.hi[j] = bx["lo"][j], bx["hi"][j]
    b.wall_mask, b.wall_mu_t, b.wall_mu_r = bx["wall_mask"], bx["wall_mu_t"], bx["wall_mu_r"]
    return b


def generator_count(gen, box, slab=(-np.inf, np.inf)):
    """Particles the generator places with lattice x in slab (host-only, no GPU)."""
    g, keep = make_generator(**gen)
    n = C.c_int64()
    st = lib().dem_generator_count(C.byref(g), C.byref(_box(box)), float(slab[0]), float(slab[1]), C.byref(n))
    if st != DEM_OK:
        raise DemError(st, "invalid generator")
    return n.value


# ---------------------------------------------------------------- bed
def _ptr(a):
    return None if a is None else a.ctypes.data


def _f64(a, shape=None):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape else a


class Bed:
    """One DEM context (one GPU).  Host arrays in, host arrays out, gid order."""

    def __init__(self, pos=None, radius=None, vel=None, angvel=None, gid=None, *, material=None, solver=None, box=None,
                 stream=None, torch_allocator=True, device=0, dist=None, generator=None):
        """dist (x-slab decomposition, include/dem.h): dict(rank, world_size, slab=(lo, hi),
        transport='nccl' with nccl_id=<128 bytes of rank 0> | 'loopback' with group=LoopbackGroup);
        pos... are then this rank's particles (inside its slab)."""
        import torch  # plumbing: stream + caching allocator
        self._torch = torch
        torch.cuda.set_device(device)
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.Stream(device=device)
        mat = dict(density=2600.0, youngs=1e7, poisson=0.3, mu_t=0.4, mu_r=0.1, restitution=0.5)
        mat.update(material or {})
        material = mat
        sol = dict(dt=1e-5, n_iter=92, n_iter_impact=0, hertz_exp=1.25, k_lin=0.0, damping_steps=4.5,
                   v_impact=-1.0, gravity=(0.0, 0.0, -9.81), rolling_dims=3, ordering=0, skin=0.0,
                   reduction=0, plate_coupling=0)
        sol.update(solver or {})
        bx = dict(lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0), wall_mask=0x3F, wall_mu_t=0.0, wall_mu_r=0.0)
        bx.update(box or {})
        desc = BedDesc()
        desc.struct_size = C.sizeof(BedDesc)
        for k, v in material.items():
            setattr(desc.mat, k, v)
        for k, v in sol.items():
            if k == "gravity":
                for j in range(3):
                    desc.solver.gravity[j] = v[j]
            else:
                setattr(desc.solver, k, v)
        for j in range(3):
            desc.box.lo[j], desc.box.hi[j] = bx["lo"][j], bx["hi"][j]
        desc.box.wall_mask, desc.box.wall_mu_t, desc.box.wall_mu_r = bx["wall_mask"], bx["wall_mu_t"], bx["wall_mu_r"]
        if generator is not None:       # on-device generator (dem_generator): no particle arrays
            desc.source = 1
            desc.gen, self._gen_keep = make_generator(**generator)
            pos, radius = np.zeros((0, 3)), np.zeros(0)
        pos = _f64(pos, (-1, 3))
        radius = _f64(radius)
        n = len(radius)
        vel, angvel = _f64(vel, (-1, 3)), _f64(angvel, (-1, 3))
        gid = None if gid is None else np.ascontiguousarray(gid, dtype=np.uint32)
        self._keep = (pos, radius, vel, angvel, gid)
        desc.parts.n = n
        desc.parts.pos, desc.parts.radius = _ptr(pos), _ptr(radius)
        desc.parts.vel, desc.parts.angvel, desc.parts.gid = _ptr(vel), _ptr(angvel), _ptr(gid)
        desc.parts.on_device = 0
        dcfg = dist
        dist = DistDesc()
        dist.rank, dist.world_size = 0, 1
        if dcfg:                   # decomposed (world_size 1 with a transport: the transport self-test)
            dist.rank, dist.world_size = int(dcfg["rank"]), int(dcfg["world_size"])
            self._world = dist.world_size
            dist.slab_lo, dist.slab_hi = float(dcfg["slab"][0]), float(dcfg["slab"][1])
            if dcfg.get("transport", "nccl") == "loopback":
                dist.transport, dist.loopback = 1, dcfg["group"].handle
                self._group = dcfg["group"]
            else:
                self._nccl_id = (C.c_ubyte * 128).from_buffer_copy(dcfg["nccl_id"])
                dist.transport, dist.nccl_unique_id = 0, C.cast(self._nccl_id, C.c_void_p)
        dist.cuda_stream = self.stream.cuda_stream
        if torch_allocator:
            dev, strm = device, self.stream.cuda_stream

            def _alloc(nbytes, _ctx):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), dev, strm)
                except Exception:   # OOM -> the library reports DEM_ERR_OOM
                    return None

            def _free(ptr, _ctx):
                torch.cuda.caching_allocator_delete(ptr)

            self._alloc_cb, self._free_cb = ALLOC_FN(_alloc), FREE_FN(_free)
            dist.alloc, dist.free = self._alloc_cb, self._free_cb
        self.n = n
        self.material, self.solver, self.box = material, sol, bx
        h = C.c_void_p()
        st = lib().dem_create_bed(C.byref(desc), C.byref(dist), C.byref(h))
        if st != DEM_OK:
            raise DemError(st, lib().dem_last_error(None).decode())
        self._h = h
        if getattr(self, "_group", None) is not None:
            self._group._beds.add(self)
        self.last_report = None
        if generator is not None:
            self.n = self.n_owned

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib().dem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != DEM_OK:
            msg = lib().dem_last_error(self._h).decode()
            raise (DivergedError if st == DEM_ERR_DIVERGED else DemError)(st, msg)

    # -- stepping
    def step(self, n=1):
        rep = StepReport()
        self._check(lib().dem_step(self._h, int(n), C.byref(rep)))
        self.last_report = rep.as_dict()
        return self.last_report

    def set_solver(self, **kw):
        """Replace solver settings (keys of dem_solver); unspecified keys keep their values.  The
        mirror (self.solver) changes only once the library accepted the new settings."""
        merged = dict(self.solver)
        merged.update(kw)
        s = Solver()
        for k, v in merged.items():
            if k == "gravity":
                for j in range(3):
                    s.gravity[j] = v[j]
            else:
                setattr(s, k, v)
        self._check(lib().dem_set_solver(self._h, C.byref(s)))
        self.solver = merged

    @property
    def n_owned(self):
        """Particles this rank owns now (all of them with world_size 1)."""
        return int(lib().dem_num_particles(self._h))

    @property
    def n_local(self):
        return int(lib().dem_num_local(self._h))

    # -- state
    def get_state(self):
        n = self.n_owned
        out = {k: np.empty((n, 3)) for k in ("pos", "vel", "angvel")}
        out["radius"] = np.empty(n)
        out["gid"] = np.empty(n, dtype=np.uint32)
        v = StateView(n, *(_ptr(out[k]) for k in ("pos", "vel", "angvel", "radius", "gid")), 0, 0)
        self._check(lib().dem_get_state(self._h, C.byref(v)))
        return out

    def get_state_device(self, out):
        """out: dict of torch CUDA tensors pos/vel/angvel (cap,3) float64, radius (cap,) f64, gid (cap,)
        int32 with cap >= n_owned; fills the first n_owned rows (gid order) and returns n_owned."""
        cap = min(int(t.shape[0]) for t in out.values())
        v = StateView(cap, *(out[k].data_ptr() if k in out else None for k in ("pos", "vel", "angvel", "radius", "gid")), 1, 0)
        self._check(lib().dem_get_state(self._h, C.byref(v)))
        return int(v.n)

    def get_state_into(self, out):
        """Host variant of get_state_device: out = dict of caller-owned HOST arrays (numpy, or torch
        CPU tensors, e.g. pinned) pos/vel/angvel (cap,3) f64 and optionally radius (cap,) f64, gid
        (cap,) u32 with cap >= n_owned; dem_get_state copies into them.  Returns n_owned."""
        def addr(t):
            return t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data
        cap = min(int(t.shape[0]) for t in out.values())
        v = StateView(cap, *(addr(out[k]) if k in out else None for k in ("pos", "vel", "angvel", "radius", "gid")), 0, 0)
        self._check(lib().dem_get_state(self._h, C.byref(v)))
        return int(v.n)

    def set_state(self, pos, radius, vel=None, angvel=None, gid=None, hist=None):
        pos, radius = _f64(pos, (-1, 3)), _f64(radius)
        vel, angvel = _f64(vel, (-1, 3)), _f64(angvel, (-1, 3))
        gid = None if gid is None else np.ascontiguousarray(gid, dtype=np.uint32)
        v = StateView(len(radius), _ptr(pos), _ptr(vel), _ptr(angvel), _ptr(radius), _ptr(gid), 0, 0)
        hv = None
        if hist is not None and len(hist):
            keys = np.ascontiguousarray(hist["key"], dtype=np.uint64)
            P = np.ascontiguousarray(hist["P"], dtype=np.float64)
            self._hk = (keys, P)
            hv = ContactView(len(keys), keys.ctypes.data, None, None, P.ctypes.data, 0, 0)
        self._check(lib().dem_set_state(self._h, C.byref(v), C.byref(hv) if hv is not None else None))

    def get_contacts(self):
        v = ContactView(0, None, None, None, None, 0, 0)
        st = lib().dem_get_contacts(self._h, C.byref(v))
        if st == DEM_ERR_INVALID and v.n > 0:
            pass
        elif st != DEM_OK:
            self._check(st)
        n = v.n
        out = np.zeros(n, dtype=CONTACT_DTYPE)
        if n == 0:
            return out
        key = np.empty(n, dtype=np.uint64)
        nrm = np.empty((n, 3))
        dl = np.empty(n)
        P = np.empty((n, 7))
        v = ContactView(n, key.ctypes.data, nrm.ctypes.data, dl.ctypes.data, P.ctypes.data, 0, 0)
        self._check(lib().dem_get_contacts(self._h, C.byref(v)))
        out["key"], out["n"], out["delta"], out["P"] = key, nrm, dl, P
        return out

    def get_forces(self):
        n = self.n_owned
        F = np.empty((n, 3))
        T = np.empty((n, 3))
        self._check(lib().dem_get_forces(self._h, F.ctypes.data, T.ctypes.data, 0))
        return F, T

    # -- boundaries
    def add_plate(self, boxes_lo, boxes_hi, pos, mass, mu_t=0.4, mu_r=0.1):
        self.n_plates = getattr(self, "n_plates", 0) + 1
        lo = np.ascontiguousarray(boxes_lo, dtype=np.float64).reshape(-1, 3)
        hi = np.ascontiguousarray(boxes_hi, dtype=np.float64).reshape(-1, 3)
        d = PlateDesc(len(lo), 0, lo.ctypes.data, hi.ctypes.data, mass, mu_t, mu_r)
        p = (C.c_double * 3)(*pos)
        pid = C.c_int32()
        self._check(lib().dem_add_plate(self._h, C.byref(d), p, C.byref(pid)))
        return pid.value

    def drive_plate(self, plate, axis, mode, target, ramp_time=0.0, f_min=-np.inf, f_max=np.inf):
        """Drive one plate axis (dem_drive_plate): f_min/f_max limit a velocity axis' motor force (Eq. 4)."""
        self._check(lib().dem_drive_plate(self._h, plate, axis, mode, target, ramp_time, f_min, f_max))

    def get_plate(self, plate):
        s = PlateState()
        self._check(lib().dem_get_plate(self._h, plate, C.byref(s)))
        return {"pos": list(s.pos), "vel": list(s.vel), "force": list(s.force),
                "motor_force": list(s.motor_force), "n_contacts": s.n_contacts}

    def add_particles(self, pos, radius, vel=None, angvel=None, gid=None):
        """dem_add_particles (single context): append particles, keeping state and contact history."""
        pos, radius = _f64(pos, (-1, 3)), _f64(radius)
        vel, angvel = _f64(vel, (-1, 3)), _f64(angvel, (-1, 3))
        gid = np.ascontiguousarray(gid, dtype=np.uint32)
        self._check(lib().dem_add_particles(self._h, len(radius), _ptr(pos), _ptr(radius), _ptr(vel), _ptr(angvel),
                                            _ptr(gid), 0))
        self.n = self.n_owned

    def remove_particles(self, axis, lo, hi):
        """dem_remove_particles (single context): drop particles with x[axis] outside [lo, hi];
        returns how many were removed."""
        out = C.c_int64()
        self._check(lib().dem_remove_particles(self._h, int(axis), float(lo), float(hi), C.byref(out)))
        self.n = self.n_owned
        return out.value

    def rebalance(self, n_bins=1024, world_size=None):
        """dem_rebalance (collective): slab faces toward particle-count quantiles; returns the
        new interior faces (world_size - 1 values; [] without a decomposition)."""
        g = world_size or getattr(self, "_world", 1)
        out = (C.c_double * max(g - 1, 1))()
        self._check(lib().dem_rebalance(self._h, int(n_bins), out))
        return list(out)[: g - 1]

    def get_wall(self, wall):
        """dem_get_wall: plane point, inward normal, normal velocity, contact reaction [N]."""
        s = WallState()
        self._check(lib().dem_get_wall(self._h, wall, C.byref(s)))
        return {"point": list(s.point), "normal": list(s.normal), "velocity": s.velocity, "force": list(s.force),
                "n_contacts": s.n_contacts}

    def drive_wall(self, wall, normal_velocity):
        self._check(lib().dem_drive_wall(self._h, wall, normal_velocity))

    # -- timing
    def set_timing(self, on=True):
        self._check(lib().dem_set_timing(self._h, int(on)))

    def reset_timing(self):
        self._check(lib().dem_reset_timing(self._h))

    def bench_sweeps(self, variant, n):
        """Diagnostic: (ms per sweep, max relative |dv| vs the shipped kernel) of a sweep variant."""
        ms, dv = C.c_double(), C.c_double()
        self._check(lib().dem_bench_sweeps(self._h, variant, n, C.byref(ms), C.byref(dv)))
        return ms.value, dv.value

    def timing(self):
        t = Timing()
        self._check(lib().dem_get_timing(self._h, C.byref(t)))
        return t.as_dict()
