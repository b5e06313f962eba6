"""fp64 CPU oracle for the nonsmooth-DEM step of arXiv 2501.05300 — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product (``paper_2501_05300_b200``)
never imports it and shares no code with it.

This module is a ctypes marshalling layer over ``liboracle.so`` (built from
``dem_oracle.c`` by :func:`build`); all arithmetic lives in the C file, which cites the
paper passage each function follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "dem_oracle.c")

WALL_KEY_BASE = 0xFFFFFFF0  # 2^32-16+w
PLATE_KEY_BASE = 0xFFFFF000  # 2^32-4096+16p+b
MAX_BOX = 8


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc, fp64, no FMA contraction."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
        os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-o", LIB, SRC, "-lm"]
        )
    return LIB


class Params(C.Structure):
    _fields_ = [
        ("rho", C.c_double), ("E", C.c_double), ("nu", C.c_double),
        ("mu_t", C.c_double), ("mu_r", C.c_double), ("e_rest", C.c_double),
        ("h", C.c_double), ("n_it", C.c_int32), ("n_imp", C.c_int32),
        ("e_H", C.c_double), ("k_lin", C.c_double), ("damp_steps", C.c_double),
        ("v_imp", C.c_double), ("g", C.c_double * 3),
        ("rolling_dims", C.c_int32), ("ordering", C.c_int32),
        ("plate_coupling", C.c_int32), ("pad", C.c_int32),
    ]


class Wall(C.Structure):
    _fields_ = [("p", C.c_double * 3), ("n", C.c_double * 3), ("vel", C.c_double),
                ("mu_t", C.c_double), ("mu_r", C.c_double), ("id", C.c_int32), ("pad", C.c_int32)]


class Plate(C.Structure):
    _fields_ = [
        ("nbox", C.c_int32), ("pad", C.c_int32),
        ("lo", (C.c_double * 3) * MAX_BOX), ("hi", (C.c_double * 3) * MAX_BOX),
        ("pos", C.c_double * 3), ("vel", C.c_double * 3),
        ("mass", C.c_double), ("mu_t", C.c_double), ("mu_r", C.c_double),
        ("mode", C.c_int32 * 3), ("pad2", C.c_int32),
        ("target", C.c_double * 3), ("ramp", C.c_double * 3), ("t0", C.c_double * 3),
        ("force", C.c_double * 3),
        ("limit", C.c_int32 * 3), ("pad3", C.c_int32),
        ("fmin", C.c_double * 3), ("fmax", C.c_double * 3), ("motor", C.c_double * 3),
    ]


class Contact(C.Structure):
    _fields_ = [("key", C.c_uint64), ("n", C.c_double * 3), ("delta", C.c_double),
                ("P", C.c_double * 7)]


class World(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("x", C.POINTER(C.c_double)), ("v", C.POINTER(C.c_double)), ("w", C.POINTER(C.c_double)),
        ("r", C.POINTER(C.c_double)), ("gid", C.POINTER(C.c_uint32)),
        ("n_walls", C.c_int32), ("n_plates", C.c_int32),
        ("walls", C.POINTER(Wall)), ("plates", C.POINTER(Plate)),
        ("time", C.c_double),
    ]


class Report(C.Structure):
    _fields_ = [
        ("n_contacts", C.c_int64), ("n_pp", C.c_int64), ("n_wall", C.c_int64),
        ("n_plate", C.c_int64), ("n_degenerate", C.c_int64),
        ("impact_fired", C.c_int32), ("pad", C.c_int32),
        ("ke", C.c_double), ("max_v", C.c_double),
        ("max_normal_residual", C.c_double), ("max_cone_excess", C.c_double),
    ]


CONTACT_DTYPE = np.dtype([("key", "<u8"), ("n", "<f8", (3,)), ("delta", "<f8"), ("P", "<f8", (7,))])
assert CONTACT_DTYPE.itemsize == C.sizeof(Contact)

_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        d, i32, i64 = C.c_double, C.c_int32, C.c_int64
        pd = C.POINTER(C.c_double)
        L.or_mass_inertia.argtypes = [d, d, pd, pd]
        L.or_contact_params.argtypes = [d, d, d, d, d, d, d, pd, pd, pd, pd]
        L.or_profile_diameter.argtypes = [d, d, d, d]
        L.or_profile_diameter.restype = d
        L.or_layer_schedule.argtypes = [d, d, d, d, pd, pd, i32]
        L.or_layer_schedule.restype = i32
        L.or_contact_network_length.argtypes = [d, d, d, d, d]
        L.or_contact_network_length.restype = d
        L.or_solver_iterations.argtypes = [d, d]
        L.or_solver_iterations.restype = i32
        L.or_planned_timestep.argtypes = [d, d, d, d]
        L.or_planned_timestep.restype = d
        L.or_detect.argtypes = [C.POINTER(World), C.POINTER(Params), C.c_void_p, i64,
                                C.POINTER(i64), C.POINTER(i64)]
        L.or_detect.restype = i32
        L.or_contacts_of.argtypes = [C.POINTER(World), C.c_void_p, i64, C.c_void_p, i64, C.POINTER(i64)]
        L.or_contacts_of.restype = i32
        L.or_step.argtypes = [C.POINTER(World), C.POINTER(Params), C.c_void_p, i64, C.c_void_p, i64,
                              C.POINTER(i64), pd, pd, C.POINTER(Report)]
        L.or_step.restype = i32
        L.or_color_contacts.argtypes = [i64, C.c_void_p, C.c_void_p, C.c_void_p, i64, C.c_void_p]
        L.or_color_contacts.restype = i32
        L.or_splitmix64.argtypes = [C.c_uint64]
        L.or_splitmix64.restype = C.c_uint64
        L.or_set_binning.argtypes = [i32]
        L.or_set_binning.restype = None
        L.or_set_threads.argtypes = [i32]
        L.or_set_threads.restype = i32
        _lib = L
    return _lib


def set_binning(on: bool) -> None:
    """SURVEY §8(c) binning mode: particle pairs from a uniform cell list (identical contact set
    and order as the brute force, pinned in tests/test_oracle_pins.py); for big-bed timing."""
    lib().or_set_binning(1 if on else 0)


def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's sweeps (n <= 0: query); returns the count in effect.  The
    results are bit-identical for any count (pinned in tests/test_oracle_pins.py)."""
    return int(lib().or_set_threads(int(n)))


# ----------------------------------------------------------------------------- pure helpers

def color_contacts(key, a, b, n_particles):
    """Greedy colouring of the contact conflict graph in decreasing splitmix64(key) priority
    (or_color_contacts).  Returns (colours array, number of colours)."""
    key = np.ascontiguousarray(key, dtype=np.uint64)
    a = np.ascontiguousarray(a, dtype=np.int64)
    b = np.ascontiguousarray(b, dtype=np.int64)
    col = np.empty(len(key), dtype=np.int32)
    n = lib().or_color_contacts(len(key), key.ctypes.data, a.ctypes.data, b.ctypes.data, int(n_particles),
                                col.ctypes.data)
    return col, n


def splitmix64(x):
    return int(lib().or_splitmix64(int(x)))


def mass_inertia(d: float, rho: float):
    m, I = C.c_double(), C.c_double()
    lib().or_mass_inertia(d, rho, C.byref(m), C.byref(I))
    return m.value, I.value


def contact_params(da, db, Ea, Eb, nua, nub, e_H=1.25):
    out = [C.c_double() for _ in range(4)]
    lib().or_contact_params(da, db, Ea, Eb, nua, nub, e_H, *[C.byref(o) for o in out])
    return tuple(o.value for o in out)  # E*, d*, k_n, eps_n


def profile_diameter(d_min, d_max, gamma, depth):
    return lib().or_profile_diameter(d_min, d_max, gamma, depth)


def layer_schedule(d_min, d_max, r, eta, cap=256):
    d = (C.c_double * cap)()
    z = (C.c_double * cap)()
    n = lib().or_layer_schedule(d_min, d_max, r, eta, d, z, cap)
    return np.array(d[:n]), np.array(z[:n])


def contact_network_length(d_min, d_max, r, eta, h):
    return lib().or_contact_network_length(d_min, d_max, r, eta, h)


def solver_iterations(n_d, eps):
    return lib().or_solver_iterations(n_d, eps)


def planned_timestep(d, eps, rho, sigma):
    return lib().or_planned_timestep(d, eps, rho, sigma)


# ----------------------------------------------------------------------------- world wrapper

def make_params(**kw) -> Params:
    """Defaults: BASELINE.json configs' material (rho 2600, E 10 MPa, nu .3, mu .4/.1, e .5)."""
    p = Params()
    p.rho, p.E, p.nu = kw.get("rho", 2600.0), kw.get("E", 1e7), kw.get("nu", 0.3)
    p.mu_t, p.mu_r, p.e_rest = kw.get("mu_t", 0.4), kw.get("mu_r", 0.1), kw.get("e_rest", 0.5)
    p.h = kw.get("h", 1e-5)
    p.n_it, p.n_imp = kw.get("n_it", 92), kw.get("n_imp", 0)
    p.e_H, p.k_lin = kw.get("e_H", 1.25), kw.get("k_lin", 0.0)
    p.damp_steps = kw.get("damp_steps", 4.5)
    p.v_imp = kw.get("v_imp", -1.0)
    g = kw.get("g", (0.0, 0.0, -9.81))
    for k in range(3):
        p.g[k] = g[k]
    p.rolling_dims = kw.get("rolling_dims", 3)
    p.ordering = kw.get("ordering", 0)          # 0 Jacobi (R2), 1 coloured Gauss-Seidel (NEXT-1)
    p.plate_coupling = kw.get("plate_coupling", 0)   # 0 staggered (R18), 1 monolithic (R18b)
    return p


def box_walls(lo, hi, mask=0x3F, mu_t=0.0, mu_r=0.0):
    """Six axis-aligned walls of the box [lo, hi] (inward normals); order -x,+x,-y,+y,-z,+z."""
    walls = []
    for ax in range(3):
        for side in range(2):
            if not (mask >> (2 * ax + side)) & 1:
                continue
            w = Wall()
            p = [0.0, 0.0, 0.0]
            n = [0.0, 0.0, 0.0]
            p[ax] = lo[ax] if side == 0 else hi[ax]
            n[ax] = 1.0 if side == 0 else -1.0
            for k in range(3):
                w.p[k], w.n[k] = p[k], n[k]
            w.vel, w.mu_t, w.mu_r = 0.0, mu_t, mu_r
            w.id = 2 * ax + side
            walls.append(w)
    return walls


def make_plate(boxes_lo, boxes_hi, pos, mass, mu_t=0.4, mu_r=0.1) -> Plate:
    P = Plate()
    P.nbox = len(boxes_lo)
    assert P.nbox <= MAX_BOX
    for b in range(P.nbox):
        for k in range(3):
            P.lo[b][k], P.hi[b][k] = boxes_lo[b][k], boxes_hi[b][k]
    for k in range(3):
        P.pos[k] = pos[k]
        P.vel[k] = 0.0
    P.mass, P.mu_t, P.mu_r = mass, mu_t, mu_r
    return P


class OracleWorld:
    """Holds numpy state and runs oracle steps on it (fp64, caller order = gid order)."""

    def __init__(self, x, v, w, r, gid, walls=(), plates=(), time=0.0):
        self.x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3).copy()
        self.v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 3).copy()
        self.w = np.ascontiguousarray(w, dtype=np.float64).reshape(-1, 3).copy()
        self.r = np.ascontiguousarray(r, dtype=np.float64).copy()
        self.gid = np.ascontiguousarray(gid, dtype=np.uint32).copy()
        self.walls = (Wall * max(1, len(walls)))(*walls)
        self.n_walls = len(walls)
        self.plates = (Plate * max(1, len(plates)))(*plates)
        self.n_plates = len(plates)
        self.time = time
        self.hist = np.zeros(0, dtype=CONTACT_DTYPE)
        self.last_report = None

    def _world(self) -> World:
        W = World()
        W.n = len(self.r)
        dp = C.POINTER(C.c_double)
        W.x = self.x.ctypes.data_as(dp)
        W.v = self.v.ctypes.data_as(dp)
        W.w = self.w.ctypes.data_as(dp)
        W.r = self.r.ctypes.data_as(dp)
        W.gid = self.gid.ctypes.data_as(C.POINTER(C.c_uint32))
        W.n_walls, W.n_plates = self.n_walls, self.n_plates
        W.walls = C.cast(self.walls, C.POINTER(Wall))
        W.plates = C.cast(self.plates, C.POINTER(Plate))
        W.time = self.time
        return W

    def detect(self, params: Params | None = None):
        params = params or make_params()
        W = self._world()
        cap = max(1024, 64 * len(self.r) + 64)
        out = np.zeros(cap, dtype=CONTACT_DTYPE)
        n, nd = C.c_int64(), C.c_int64()
        rc = lib().or_detect(C.byref(W), C.byref(params), out.ctypes.data, cap, C.byref(n), C.byref(nd))
        if rc:
            raise RuntimeError(f"or_detect failed rc={rc}")
        return out[: n.value].copy(), nd.value

    def contacts_of(self, idx):
        """Brute-force contacts of the given particle indices (caller order), sorted by key."""
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        W = self._world()
        cap = 64 * len(idx) + 64
        out = np.zeros(cap, dtype=CONTACT_DTYPE)
        n = C.c_int64()
        rc = lib().or_contacts_of(C.byref(W), idx.ctypes.data, len(idx), out.ctypes.data, cap, C.byref(n))
        if rc:
            raise RuntimeError("or_contacts_of failed")
        return out[: n.value].copy()

    def step(self, params: Params, n_steps: int = 1, want_forces: bool = False):
        """Advance n_steps; returns (contacts of the last step, F, T)."""
        F = np.zeros((len(self.r), 3)) if want_forces else None
        T = np.zeros((len(self.r), 3)) if want_forces else None
        out = None
        for _ in range(n_steps):
            W = self._world()
            cap = max(1024, 64 * len(self.r) + 64)
            out = np.zeros(cap, dtype=CONTACT_DTYPE)
            n = C.c_int64()
            rep = Report()
            dp = C.POINTER(C.c_double)
            rc = lib().or_step(
                C.byref(W), C.byref(params), self.hist.ctypes.data if len(self.hist) else None,
                len(self.hist), out.ctypes.data, cap, C.byref(n),
                F.ctypes.data_as(dp) if F is not None else None,
                T.ctypes.data_as(dp) if T is not None else None, C.byref(rep))
            if rc == -1:
                raise RuntimeError("or_step: contact capacity exceeded")
            if rc == -3:
                raise RuntimeError("or_step: the Gauss-Seidel colouring needs more than 256 colours")
            self.time = W.time
            out = out[: n.value].copy()
            self.hist = out
            self.last_report = rep
            if rc == -2:
                raise FloatingPointError("or_step: NaN/Inf in state")
        return out, F, T
