"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on identical inputs.

Bars (BASELINE.json acceptance): contact pair set bit-exact; per-particle force and torque
relative error <= 1e-5 under the physical floors of tests/parity.py (reading R34)."""
import numpy as np
import pytest

import synth
from tests.parity import compare_step

pytestmark = pytest.mark.gpu

TOL_F = 1e-5


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_one_step_random_cloud(seed):
    bed = synth.random_cloud(600, (0, 0, 0), (0.05, 0.05, 0.05), 1.5e-3, 3.5e-3, seed, v_scale=0.02, w_scale=2.0)
    res = compare_step(bed, n_it=40, dt=1e-5)
    assert res["pairs_equal"], res
    assert res["force_err"] <= TOL_F and res["torque_err"] <= TOL_F, res


def test_one_step_polydisperse_8x_multilevel():
    bed = synth.random_cloud(800, (0, 0, 0), (0.08, 0.08, 0.08), 1e-3, 8e-3, 9, v_scale=0.01, loguniform=True)
    res = compare_step(bed, n_it=40, dt=1e-5)
    assert res["pairs_equal"], res
    assert res["force_err"] <= TOL_F and res["torque_err"] <= TOL_F, res


def test_config0_first_steps():
    bed = synth.config0()
    res = compare_step(bed, n_it=92, dt=1e-5, n_steps=3)
    assert res["pairs_equal"], res
    assert res["force_err"] <= TOL_F and res["torque_err"] <= TOL_F, res
