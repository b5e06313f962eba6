"""SURVEY §8(d) mini-bed plate-curve protocols (acceptance criterion 4: "plate pressure-sinkage and
shear stress-displacement curves agree within 2 % RMS normalised error").  Test infrastructure:
the protocol definitions shared by the ORACLE side (tests/fixtures/make_curves_mini.py, run once
on the CPU; it writes the settled beds and the oracle curves under tests/golden/) and the GPU
side (tests/test_gpu_z_curves_mini.py).  Nothing here holds arithmetic of the method: it places
spheres (synth), places a plate, and filters curves.

c1-mini (config 1 shape, P:205-217 pressure-sinkage): 0.1 x 0.1 x 0.075 m box, 2 mm spheres over
the top 0.015 m and 4 mm below (+-10 %); a 25 mm square flat plate pressed down
kinematically at 0.05 m/s for 0.01 m: 4e4 steps of 5e-6 s, N_it = 50; curve = plate reaction F_z.

c2-mini (config 2 shape, P:254 shear): 0.25 x 0.125 x 0.125 m box, radius growing linearly with
depth from 2 mm at the surface to 5.5 mm at the bottom (Eq. 1); the paper's grouser plate
scaled by 1/4 (75 mm long, 4 grousers 10.75 mm deep x 6.4 mm long at an 18.75 mm pitch,
100 mm wide) on a force-driven vertical axis carrying 10 kPa over its footprint (75 N), sheared
along x at 0.02 m/s (ramped over 10 ms) for 5 mm: 5e4 steps of 5e-6 s, N_it = 50; curve = the
shear reaction F_x.

Both start from a bed settled under gravity by the oracle (h = 1e-4 s, 30 sweeps) with its
contact history, the plate 0.1 mm above the highest sphere under its footprint.
Error: RMS of the difference of the two curves after a 2 ms moving average, divided by the
oracle curve's maximum |value| (SURVEY §8(c) "plate curves"); the bar applies to the mean over
three seeds.
"""
from __future__ import annotations

import numpy as np

import synth

DT = 5e-6
N_IT = 50
SEEDS = (1001, 2001, 3001)
AVG_STEPS = int(round(2e-3 / DT))        # 2 ms moving average
SETTLE = dict(h=1e-4, n_it=30, steps=2500)
KINDS = ("c1", "c2")
N_STEPS = {"c1": 40000, "c2": 50000}


def make_bed(kind: str, seed: int) -> synth.Bed:
    if kind == "c1":
        return synth.banded_bed((0.1, 0.1, 0.075), [(0.0, 0.015, 2e-3), (0.015, 0.075, 4e-3)], seed, spacing=2.25,
                                name="c1-mini")
    if kind == "c2":
        return synth.graded_bed((0.25, 0.125, 0.125), 2e-3, 5.5e-3, 0.125, seed, spacing=2.25, name="c2-mini")
    raise ValueError(kind)


WALL_MASK = 0x0F | 0x10          # side walls and the floor; open top (the plate comes from above)


def plate(kind: str, x: np.ndarray, r: np.ndarray, box_hi):
    """(boxes_lo, boxes_hi, start pos, mass, drives): drives = list of (axis, mode, target, ramp)
    with mode 1 = kinematic velocity, 2 = force (include/dem.h dem_axis_mode)."""
    if kind == "c1":
        hx = hy = 0.0125
        lo, hi = [(-hx, -hy, 0.0)], [(hx, hy, 0.005)]
        tip = 0.0
        drives = [(2, 1, -0.05, 0.0)]
    else:
        hx, hy = 0.0375, 0.05
        lo, hi = [(-hx, -hy, 0.0)], [(hx, hy, 0.005)]
        for k in range(4):
            xc = -hx + 0.009375 + 0.01875 * k
            lo.append((xc - 0.0032, -hy, -0.01075))
            hi.append((xc + 0.0032, hy, 0.0))
        tip = -0.01075
        area = (2 * hx) * (2 * hy)
        drives = [(2, 2, -10e3 * area, 0.0), (0, 1, 0.02, 0.01)]
    cx, cy = 0.5 * box_hi[0], 0.5 * box_hi[1]
    m = (np.abs(x[:, 0] - cx) <= hx + r) & (np.abs(x[:, 1] - cy) <= hy + r)
    top = float((x[m, 2] + r[m]).max())
    pos = (cx, cy, top - tip + 1e-4)
    vol = sum((b[0] - a[0]) * (b[1] - a[1]) * (b[2] - a[2]) for a, b in zip(lo, hi))
    return lo, hi, pos, 7850.0 * vol, drives


def plate_coupling(kind: str) -> int:
    """c2's plate rides on a 10 kPa force axis: staggered coupling (R18) lets the 0.5 kg plate
    take each step's full rigid-body reaction and bounce (measured: its contact count falls from
    ~430 to ~5 within 0.1 s), so c2 couples it monolithically (R18b, tools in the same
    MCP).  c1's plate is kinematic: the coupling does not apply."""
    return 1 if kind == "c2" else 0


def curve_axis(kind: str) -> int:
    return 2 if kind == "c1" else 0


def smooth(a, w=AVG_STEPS):
    a = np.asarray(a, dtype=np.float64)
    k = np.ones(w) / w
    return np.convolve(a, k, mode="valid")


def rms_error(f_gpu, f_ref):
    g, r = smooth(f_gpu), smooth(f_ref)
    return float(np.sqrt(np.mean((g - r) ** 2)) / np.abs(r).max())
