"""GPU parity on a bed shaped like the bench workload.

A full-depth column of config4-geom: the three refinement bands (r = 2 mm to 0.08 m depth,
6 mm to 0.25 m, 16 mm below, +-10 % radius jitter), the bench's jammed FCC packing
(nearest-neighbour distance 2 r_nom), walls on every side; > 50,000 spheres, ~3 contacts per
sphere.  The start state is the jammed lattice relaxed by the ORACLE (10 steps of 1e-4 s with
20 sweeps), so both sides start from the same seeded state and contact history and nothing
flows from the CUDA path into the oracle.  Then both run the bench's time step (dt = 5e-6 s,
N_it = 226 from Eqs. 8 + 10) with the Newton impact stage firing:
  * step 1: contact pairs bit-exact, per-particle forces and torques <= 1e-5 (floors of
    tests/parity.py);
  * 20 steps: positions within 1e-4 of the mean radius (the trajectory bar of BASELINE.json).
"""
import numpy as np
import pytest

import oracle as O
import synth
from tests.parity import compare_step

pytestmark = pytest.mark.gpu

BANDS = [(0.0, 0.08, 2e-3), (0.08, 0.25, 6e-3), (0.25, 0.6, 16e-3)]
N_IT = 226          # Eqs. 8 + 10 on the bands, eps = 0.02 (bench.py)


def relaxed_column():
    b = synth.banded_bed((0.17, 0.17, 0.6), BANDS, 1904, spacing=2.0, name="config4-column")
    O.set_binning(True)
    try:
        W = O.OracleWorld(b.x, b.v, b.w, b.r, b.gid, walls=O.box_walls(b.box_lo, b.box_hi))
        W.step(O.make_params(h=1e-4, n_it=20), 10)
    finally:
        O.set_binning(False)
    bed = synth.Bed(x=W.x.copy(), r=b.r, v=W.v.copy(), w=W.w.copy(), gid=b.gid, box_lo=b.box_lo,
                    box_hi=b.box_hi, name="config4-column-relaxed")
    return bed, W.hist.copy()


@pytest.fixture(scope="module")
def column():
    return relaxed_column()


def test_bench_column_one_step_forces(column):
    bed, hist = column
    assert bed.n > 50000
    O.set_binning(True)
    try:
        res = compare_step(bed, n_it=N_IT, dt=5e-6, hist=hist)
    finally:
        O.set_binning(False)
    print({k: v for k, v in res.items() if k != "detail"})
    assert res["n_contacts_ref"] > 2.5 * bed.n
    assert res["impact_ref"] == 1 and res["impact_gpu"] == 1
    assert res["pairs_equal"], res
    assert res["force_err"] <= 1e-5 and res["torque_err"] <= 1e-5, res


def test_bench_column_20_steps_positions(column):
    bed, hist = column
    O.set_binning(True)
    try:
        res = compare_step(bed, n_it=N_IT, dt=5e-6, hist=hist, n_steps=20)
    finally:
        O.set_binning(False)
    print({k: v for k, v in res.items() if k != "detail"})
    assert res["pairs_equal"], res
    assert res["x_err"] <= 1e-4 * bed.r.mean(), res
    assert res["force_err"] <= 1e-5 and res["torque_err"] <= 1e-5, res
