"""Plate curves at the SURVEY §8(d) mini-bed scale, GPU vs oracle (BASELINE.json acceptance 4:
"plate pressure-sinkage and shear stress-displacement curves agree within 2% RMS normalised
error").  Protocols in tests/curves_mini.py: c1-mini (25 mm plate pressed
0.01 m at 0.05 m/s, 4e4 steps) and c2-mini (grouser plate under 10 kPa sheared 5 mm at
0.02 m/s, 5e4 steps), N_it = 50, three seeds each.

The bar is taken on the seed-averaged curves ("mini beds, smoothing and seed
averages"; the paper repeats every case and compares means): RMS of the difference of the
GPU's and the oracle's mean curves after the 2 ms moving average, over the oracle mean curve's
maximum, <= 2 %.  The granular bed is chaotic: the two fp64 trajectories separate from rounding
onward, so single-seed curves differ by their fluctuations; the per-seed errors are printed and
recorded (profiles/r02_curves_mini.txt) beside the ensemble figure.

The oracle side ran once on the CPU (tests/fixtures/make_curves_mini.py, OpenMP oracle) and
stored its curves and the oracle-settled beds; this test loads each settled bed (or re-settles it
with the oracle when the cache is absent), checks the digest of the settled state against the one
stored with the oracle curve (both sides start from the identical state and contact history),
runs the GPU through the C-ABI, and compares the 2 ms moving averages: RMS of the difference of the
seed-averaged curves over the oracle mean curve's maximum <= 2 %.  (The file name sorts last: the
long acceptance runs come after the parity suites under `pytest -x`.)
"""
import os

import numpy as np
import pytest

import oracle as O
from tests import curves_mini as CM
from tests.fixtures.make_curves_mini import digest, settled

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
HERE = os.path.dirname(os.path.abspath(__file__))
TOL_RMS = 0.02


def gpu_curve(kind, b, W):
    from paper_2501_05300_b200 import dem
    box = dict(lo=b.box_lo, hi=b.box_hi, wall_mask=CM.WALL_MASK)
    g = dem.Bed(W.x, W.r, W.v, W.w, W.gid, solver=dict(dt=CM.DT, n_iter=CM.N_IT, plate_coupling=CM.plate_coupling(kind)),
                box=box)
    try:
        g.set_state(W.x, W.r, W.v, W.w, W.gid, hist=W.hist)
        lo, hi, pos, mass, drives = CM.plate(kind, W.x, W.r, b.box_hi)
        pid = g.add_plate(lo, hi, pos, mass)
        for ax, mode, target, ramp in drives:
            g.drive_plate(pid, ax, mode, target, ramp)
        ax = CM.curve_axis(kind)
        n = CM.N_STEPS[kind]
        f = np.empty(n)
        x = np.empty(n)
        for s in range(n):
            g.step(1)
            st = g.get_plate(pid)
            f[s] = st["force"][ax]
            x[s] = st["pos"][ax]
        return f, x
    finally:
        g.close()


@pytest.mark.parametrize("kind", CM.KINDS)
def test_plate_curve_mini_within_2pct(kind):
    O.set_threads(os.cpu_count() or 1)
    errs, fg, fr = [], [], []
    for seed in CM.SEEDS:
        path = os.path.join(HERE, "golden", f"curves_mini_{kind}_{seed}.npz")
        if not os.path.exists(path):
            pytest.skip(f"oracle curves not generated yet: {path}")
        ref = np.load(path)
        b, W = settled(kind, seed)
        assert digest(W) == str(ref["digest"]), "settled state differs from the oracle run's"
        f, x = gpu_curve(kind, b, W)
        f_ref = ref["force"].astype(np.float64)
        assert np.abs(f_ref).max() > 0
        e = CM.rms_error(f, f_ref)
        ex = float(np.abs(x - ref["pos"]).max())
        print(kind, seed, "rms", e, "max |dx| plate", ex, "max |F| ref", np.abs(f_ref).max(), "gpu", np.abs(f).max())
        errs.append(e)
        fg.append(f)
        fr.append(f_ref)
        if os.path.isdir("gpurun_out"):
            np.savez_compressed(f"gpurun_out/curves_mini_gpu_{kind}_{seed}.npz", force=f, pos=x)
    e_mean = CM.rms_error(np.mean(fg, axis=0), np.mean(fr, axis=0))
    print(kind, "per-seed rms", errs, "mean of per-seed", float(np.mean(errs)), "seed-averaged curves rms", e_mean)
    assert e_mean <= TOL_RMS, (e_mean, errs)
