"""Plate curves, GPU vs oracle (BASELINE.json acceptance: "plate pressure-sinkage and shear
stress-displacement curves agree within 2% RMS normalised error").

Input: the two-layer refined mini bed of tests/golden/plate_mini_state.npz (1 mm spheres over the
top 0.01 m, 2 mm below, settled by the oracle: tests/fixtures/make_plate_mini.py), shaped like
SURVEY §8(d) "c1-mini".  Both sides start from that state and its contact history and run the
same protocol independently:
  * pressure-sinkage (P:205-217 pressure-sinkage phase, config 1 drive): a 20 x 20 mm plate
    pressed down kinematically at 0.05 m/s for 2 mm; curve = plate reaction F_z(sinkage);
  * shear-displacement: the same plate on a force-driven vertical axis (5 N down) sheared
    along x at 0.05 m/s (ramped over 5 ms) for 2 mm; curve = traction F_x(displacement).
Error (SURVEY §8(c) "plate curves"): RMS over the run of the difference of the two curves after
a 0.4 ms moving average, divided by the oracle curve's maximum |value|.  Granular contact
networks are chaotic, so per-particle trajectories part ways over thousands of steps; the
curves are the aggregate the criterion bounds.
"""
import os

import numpy as np
import pytest

import oracle as O
import synth
from tests.parity import gpu_bed, oracle_params, oracle_world

pytestmark = [pytest.mark.gpu, pytest.mark.slow, pytest.mark.usefixtures("oracle_binning")]
HERE = os.path.dirname(os.path.abspath(__file__))
TOL_RMS = 0.02


def mini_bed():
    f = np.load(os.path.join(HERE, "golden", "plate_mini_state.npz"))
    bed = synth.Bed(x=f["x"], r=f["r"], v=f["v"], w=f["w"], gid=f["gid"], box_lo=tuple(f["box_lo"]),
                    box_hi=tuple(f["box_hi"]), name="plate-mini")
    hist = np.zeros(len(f["hist_key"]), dtype=O.CONTACT_DTYPE)
    hist["key"], hist["P"] = f["hist_key"], f["hist_P"]
    return bed, hist


def smooth(a, w):
    k = np.ones(w) / w
    return np.convolve(a, k, mode="valid")


def run_protocol(kind, n_steps=2000, dt=2e-5, n_it=40):
    bed, hist = mini_bed()
    top = float((bed.x[:, 2] + bed.r).max())
    lo, hi = [(-0.01, -0.01, 0.0)], [(0.01, 0.01, 0.004)]
    pos = (0.02, 0.02, top + 2e-4)
    mass = 0.05
    P = O.make_plate(lo, hi, pos=pos, mass=mass)
    if kind == "sinkage":
        P.mode[2], P.target[2], P.vel[2] = 1, -0.05, -0.05
    else:
        P.mode[2], P.target[2] = 2, -5.0
        P.mode[0], P.target[0], P.ramp[0] = 1, 0.05, 5e-3
    Wo = oracle_world(bed, plates=[P])
    Wo.hist = hist
    po = oracle_params(n_it, dt)
    gb = gpu_bed(bed, dt=dt, n_iter=n_it)
    gb.set_state(bed.x, bed.r, bed.v, bed.w, bed.gid, hist=hist)
    pid = gb.add_plate(lo, hi, pos, mass)
    if kind == "sinkage":
        gb.drive_plate(pid, 2, 1, -0.05)
    else:
        gb.drive_plate(pid, 2, 2, -5.0)
        gb.drive_plate(pid, 0, 1, 0.05, 5e-3)
    ax = 2 if kind == "sinkage" else 0
    f_ref, f_gpu, x_ref, x_gpu = [], [], [], []
    try:
        for _ in range(n_steps):
            Wo.step(po)
            gb.step(1)
            g = gb.get_plate(pid)
            f_ref.append(Wo.plates[0].force[ax])
            f_gpu.append(g["force"][ax])
            x_ref.append(Wo.plates[0].pos[ax])
            x_gpu.append(g["pos"][ax])
    finally:
        gb.close()
    return np.array(f_ref), np.array(f_gpu), np.array(x_ref), np.array(x_gpu), dt


def curve_error(f_ref, f_gpu, dt, window_s=4e-4):
    w = max(1, int(round(window_s / dt)))
    a, b = smooth(f_ref, w), smooth(f_gpu, w)
    return float(np.sqrt(np.mean((b - a) ** 2)) / np.abs(a).max())


def test_pressure_sinkage_curve_within_2pct():
    f_ref, f_gpu, z_ref, z_gpu, dt = run_protocol("sinkage")
    assert np.abs(z_gpu - z_ref).max() <= 1e-12                 # kinematic axis: the same drive
    assert np.abs(f_ref).max() > 1.0                              # the plate does load the bed
    err = curve_error(f_ref, f_gpu, dt)
    print("pressure-sinkage RMS error", err)
    assert err <= TOL_RMS


def test_shear_displacement_curve_within_2pct():
    f_ref, f_gpu, x_ref, x_gpu, dt = run_protocol("shear")
    assert x_ref[-1] - x_ref[0] > 1.5e-3                         # sheared ~2 mm
    assert np.abs(f_ref).max() > 0.5
    err = curve_error(f_ref, f_gpu, dt)
    print("shear-displacement RMS error", err)
    assert err <= TOL_RMS
