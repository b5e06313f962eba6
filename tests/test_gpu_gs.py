"""Coloured projected Gauss-Seidel ordering (solver.ordering = 1; P:134 PGS) on
the GPU against the oracle's Gauss-Seidel (oracle/dem_oracle.c sweep_gs, same colouring by
definition): pair sets, per-particle forces/torques (same bar as the Jacobi path), the number
of colours, and the convergence advantage the paper's solver choice rests on."""
import numpy as np
import pytest

import oracle as O
import synth
from tests.parity import compare_step, gpu_bed, oracle_params, oracle_world
from tests.test_gpu_parity import config0s

pytestmark = pytest.mark.gpu
TOL_F = 1e-5


def oracle_colours(contacts, bed):
    inv = {int(g): i for i, g in enumerate(bed.gid)}
    ka = (contacts["key"] >> np.uint64(32)).astype(np.int64)
    kb = (contacts["key"] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    a = np.array([inv[k] for k in ka], dtype=np.int64)
    b = np.array([inv[k] if k < O.PLATE_KEY_BASE else -1 for k in kb], dtype=np.int64)
    return O.color_contacts(contacts["key"], a, b, len(bed.r))[1]


@pytest.mark.parametrize("seed", [1, 2])
def test_one_step_gauss_seidel_random_cloud(seed):
    bed = synth.random_cloud(600, (0, 0, 0), (0.05, 0.05, 0.05), 1.5e-3, 3.5e-3, seed, v_scale=0.02, w_scale=2.0)
    res = compare_step(bed, n_it=40, dt=1e-5, ordering=1)
    assert res["pairs_equal"], res
    assert res["force_err"] <= TOL_F and res["torque_err"] <= TOL_F, res
    assert res["n_colors_gpu"] == oracle_colours(res["detail"]["c_ref"], bed)


def test_one_step_gauss_seidel_config0s_with_history():
    bed, hist = config0s()
    res = compare_step(bed, n_it=92, dt=1e-5, hist=hist, v_imp=1e30, ordering=1)
    assert res["pairs_equal"], res
    assert res["force_err"] <= TOL_F and res["torque_err"] <= TOL_F, res
    assert res["n_colors_gpu"] == oracle_colours(res["detail"]["c_ref"], bed)


def test_gauss_seidel_converges_faster_than_jacobi_on_gpu():
    """config 0s, 20 sweeps: the coloured Gauss-Seidel impulses are closer to the converged ones
    (2,000 Gauss-Seidel sweeps) than the Jacobi impulses after the same 20 sweeps."""
    bed, hist = config0s()

    def run(n_it, ordering):
        gb = gpu_bed(bed, dt=1e-5, n_iter=n_it, v_impact=1e30, ordering=ordering)
        gb.set_state(bed.x, bed.r, bed.v, bed.w, bed.gid, hist=hist)
        gb.step(1)
        c = gb.get_contacts()
        gb.close()
        return c["P"][:, 0]

    ref = run(2000, 1)
    e_j = np.abs(run(20, 0) - ref).max()
    e_g = np.abs(run(20, 1) - ref).max()
    assert e_g < 0.5 * e_j, (e_g, e_j)
