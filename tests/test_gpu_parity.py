"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on identical inputs.

Bars (BASELINE.json acceptance): contact pair set bit-exact; per-particle force and torque
relative error <= 1e-5 under the physical floors of tests/parity.py (reading R34);
1,000-step trajectories on config 0 (and the settled config 0s) within 1e-4 of the mean radius.
"""
import os

import numpy as np
import pytest

import oracle as O
import synth
from tests.parity import compare_step, gpu_bed, oracle_params, oracle_world

pytestmark = pytest.mark.gpu

TOL_F = 1e-5
HERE = os.path.dirname(os.path.abspath(__file__))


def dem():
    from paper_2501_05300_b200 import dem as D
    return D


def config0s():
    f = np.load(os.path.join(HERE, "golden", "config0s_state.npz"))
    bed = synth.Bed(x=f["x"], r=f["r"], v=f["v"], w=f["w"], gid=f["gid"], box_lo=tuple(f["box_lo"]),
                    box_hi=tuple(f["box_hi"]), name="config0s")
    hist = np.zeros(len(f["hist_key"]), dtype=O.CONTACT_DTYPE)
    hist["key"], hist["P"] = f["hist_key"], f["hist_P"]
    return bed, hist


# ------------------------------------------------------------------ one-step parity
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
    res = compare_step(synth.config0(), n_it=92, dt=1e-5, n_steps=3)
    assert res["pairs_equal"], res
    assert res["force_err"] <= TOL_F and res["torque_err"] <= TOL_F, res


@pytest.mark.parametrize("reduction", [0, 1])
def test_config0s_one_step_with_history(reduction):
    """Settled config 0 with its contact history as warm start: ~10k contacts;
    both per-particle reductions of the sweep (canonical packed chunks, contiguous chunks)."""
    bed, hist = config0s()
    res = compare_step(bed, n_it=92, dt=1e-5, hist=hist, v_imp=1e30, reduction=reduction)
    assert res["n_contacts_ref"] > 5000
    assert res["pairs_equal"], res
    assert res["force_err"] <= TOL_F and res["torque_err"] <= TOL_F, res


# ------------------------------------------------------------------ trajectories
def _trajectory(bed, hist, steps, every, n_it, dt):
    Wo = oracle_world(bed)
    po = oracle_params(n_it, dt)
    gb = gpu_bed(bed, dt=dt, n_iter=n_it)
    if hist is not None:
        Wo.hist = hist
        gb.set_state(bed.x, bed.r, bed.v, bed.w, bed.gid, hist=hist)
    order = np.argsort(bed.gid)
    worst = 0.0
    try:
        for k in range(steps // every):
            Wo.step(po, n_steps=every)
            gb.step(every)
            st = gb.get_state()
            worst = max(worst, float(np.abs(st["pos"] - Wo.x[order]).max()))
    finally:
        gb.close()
    return worst


@pytest.mark.slow
def test_trajectory_config0_1000_steps():
    bed = synth.config0()
    worst = _trajectory(bed, None, 1000, 100, 92, 1e-5)
    assert worst <= 1e-4 * bed.r.mean(), worst


@pytest.mark.slow
def test_trajectory_config0s_1000_steps():
    bed, hist = config0s()
    worst = _trajectory(bed, hist, 1000, 100, 92, 1e-5)
    assert worst <= 1e-4 * bed.r.mean(), worst


# ------------------------------------------------------------------ edge cases
def test_empty_bed():
    D = dem()
    b = D.Bed(np.zeros((0, 3)), np.zeros(0), box=dict(lo=(0, 0, 0), hi=(1, 1, 1)))
    rep = b.step(3)
    assert rep["n_contacts"] == 0 and rep["step"] == 3
    assert b.get_state()["pos"].shape == (0, 3)
    assert len(b.get_contacts()) == 0
    b.close()


def test_single_particle_free_flight_exact():
    D = dem()
    h, n = 1e-4, 200
    x0, v0 = np.array([[0.3, 0.4, 0.5]]), np.array([[0.5, -0.2, 1.0]])
    b = D.Bed(x0, [1e-3], v0, box=dict(lo=(0, 0, 0), hi=(1, 1, 1)), solver=dict(dt=h, n_iter=5))
    b.step(n)
    st = b.get_state()
    g = np.array([0, 0, -9.81])
    np.testing.assert_allclose(st["pos"], x0 + n * h * v0 + h * h * g * n * (n + 1) / 2, rtol=1e-12)
    np.testing.assert_allclose(st["vel"], v0 + n * h * g, rtol=1e-12)
    b.close()


def test_degenerate_coincident_centres_and_outside_box():
    """Coincident centres are counted and skipped; particles outside the container
    (clamped grid cells) still get the exact pair set."""
    bed = synth.random_cloud(300, (-0.01, -0.01, -0.01), (0.04, 0.04, 0.04), 1.5e-3, 3e-3, 21, v_scale=0.01)
    bed.x[5] = bed.x[7]
    bed.box_lo, bed.box_hi = (0.0, 0.0, 0.0), (0.03, 0.03, 0.03)
    res = compare_step(bed, n_it=30, dt=1e-5)
    assert res["pairs_equal"], res
    assert res["force_err"] <= TOL_F and res["torque_err"] <= TOL_F, res


def test_linear_model_and_planar_rolling():
    bed = synth.random_cloud(400, (0, 0, 0), (0.04, 0.04, 0.04), 1.5e-3, 3e-3, 31, v_scale=0.02, w_scale=1.0)
    Wo = oracle_world(bed)
    po = O.make_params(h=1e-5, n_it=30, e_H=1.0, k_lin=2e3, rolling_dims=2)
    gb = gpu_bed(bed, dt=1e-5, n_iter=30, hertz_exp=1.0, k_lin=2e3, rolling_dims=2)
    c_ref, F_ref, T_ref = Wo.step(po, want_forces=True)
    gb.step(1)
    c = gb.get_contacts()
    F, T = gb.get_forces()
    gb.close()
    from tests.parity import force_errors
    eF, eT = force_errors(F, T, F_ref, T_ref, c_ref, bed, 2600.0, 1e-5)
    assert np.array_equal(c["key"], c_ref["key"])
    assert eF.max() <= TOL_F and eT.max() <= TOL_F, (eF.max(), eT.max())


def test_newton_impact_headon():
    D = dem()
    r = 3e-3
    x = np.array([[0.05, 0.05, 0.05], [0.05 + 2 * r - 1e-10, 0.05, 0.05]])
    v = np.array([[0.3, 0, 0], [-0.1, 0, 0]])
    b = D.Bed(x, [r, r], v, box=dict(lo=(0, 0, 0), hi=(0.1, 0.1, 0.1)), material=dict(mu_t=0, mu_r=0),
              solver=dict(dt=1e-6, n_iter=20, gravity=(0, 0, 0)))
    rep = b.step(1)
    st = b.get_state()
    b.close()
    assert rep["impact_fired"] == 1
    # impulses are stored in fp32: the separation speed is exact to 2^-24 relative
    assert st["vel"][1, 0] - st["vel"][0, 0] == pytest.approx(0.5 * 0.4, rel=2.0 ** -23)
    assert st["vel"][:, 0].sum() == pytest.approx(0.2, abs=1e-15)


def _small_bed_for_plates(seed):
    b = synth.random_cloud(250, (0.002, 0.002, 0.002), (0.028, 0.028, 0.014), 1.5e-3, 2.5e-3, seed)
    b.box_lo, b.box_hi = (0.0, 0.0, 0.0), (0.03, 0.03, 0.05)
    return b


@pytest.mark.parametrize("coupling", [0, 1])
def test_plates_kinematic_and_force_axes_vs_oracle(coupling):
    """A grouser plate (3 boxes) pressed down kinematically and a flat plate on a force axis,
    20 steps on both sides: pair sets every step, plate forces and positions; the force axis
    staggered (R18) or monolithic (R18b, solver.plate_coupling = 1)."""
    bed = _small_bed_for_plates(41)
    lo = [(-0.006, -0.006, 0.0), (-0.006, -0.006, -0.003), (0.003, -0.006, -0.003)]
    hi = [(0.006, 0.006, 0.002), (-0.004, 0.006, 0.0), (0.005, 0.006, 0.0)]
    top = bed.x[:, 2].max() + 2.6e-3
    P1 = O.make_plate(lo, hi, pos=(0.009, 0.015, top), mass=0.05)
    P1.mode[2], P1.target[2], P1.vel[2] = 1, -0.05, -0.05
    P2 = O.make_plate([(-0.004, -0.004, 0.0)], [(0.004, 0.004, 0.002)], pos=(0.022, 0.015, top - 1e-3), mass=0.01)
    P2.mode[2], P2.target[2] = 2, -0.5
    Wo = oracle_world(bed, plates=[P1, P2])
    po = oracle_params(30, 1e-5, plate_coupling=coupling)
    gb = gpu_bed(bed, dt=1e-5, n_iter=30, plate_coupling=coupling)
    p1 = gb.add_plate(lo, hi, (0.009, 0.015, top), 0.05)
    gb.drive_plate(p1, 2, 1, -0.05)
    p2 = gb.add_plate([(-0.004, -0.004, 0.0)], [(0.004, 0.004, 0.002)], (0.022, 0.015, top - 1e-3), 0.01)
    gb.drive_plate(p2, 2, 2, -0.5)
    try:
        for s in range(20):
            c_ref, _, _ = Wo.step(po)
            gb.step(1)
            c = gb.get_contacts()
            assert np.array_equal(c["key"], c_ref["key"]), s
        g1, g2 = gb.get_plate(p1), gb.get_plate(p2)
    finally:
        gb.close()
    assert (c_ref["key"] & np.uint64(0xFFFFFFFF) >= np.uint64(O.PLATE_KEY_BASE)).sum() > 0
    assert g1["pos"][2] == pytest.approx(Wo.plates[0].pos[2], abs=1e-12)
    scale = max(abs(Wo.plates[0].force[2]), 1e-3)
    assert abs(g1["force"][2] - Wo.plates[0].force[2]) <= 1e-5 * scale
    assert g2["pos"][2] == pytest.approx(Wo.plates[1].pos[2], abs=1e-9)


def test_moving_wall_vs_oracle():
    bed = _small_bed_for_plates(43)
    Wo = oracle_world(bed)
    Wo.walls[1].vel = 0.2        # +x wall moving inward
    po = oracle_params(30, 1e-5)
    gb = gpu_bed(bed, dt=1e-5, n_iter=30)
    gb.drive_wall(1, 0.2)
    try:
        for s in range(30):
            c_ref, _, _ = Wo.step(po)
            gb.step(1)
        c = gb.get_contacts()
        st = gb.get_state()
    finally:
        gb.close()
    assert np.array_equal(c["key"], c_ref["key"])
    order = np.argsort(bed.gid)
    assert np.abs(st["pos"] - Wo.x[order]).max() < 1e-9


# ------------------------------------------------------------------ API behaviour
def test_determinism_bit_identical():
    bed = synth.random_cloud(2000, (0, 0, 0), (0.08, 0.08, 0.08), 1.5e-3, 4e-3, 51, v_scale=0.02, w_scale=1.0)
    outs = []
    for _ in range(2):
        gb = gpu_bed(bed, dt=1e-5, n_iter=40)
        gb.step(5)
        st = gb.get_state()
        c = gb.get_contacts()
        gb.close()
        outs.append((st, c))
    for k in ("pos", "vel", "angvel"):
        assert np.array_equal(outs[0][0][k], outs[1][0][k]), k
    assert np.array_equal(outs[0][1]["P"], outs[1][1]["P"])


def test_state_roundtrip_and_errors():
    D = dem()
    bed = synth.random_cloud(100, (0, 0, 0), (0.03, 0.03, 0.03), 1.5e-3, 3e-3, 61, v_scale=0.01)
    gb = gpu_bed(bed, dt=1e-5, n_iter=10)
    with pytest.raises(D.DemError) as e:
        gb.get_forces()
    assert e.value.status == D.DEM_ERR_STATE
    st = gb.get_state()
    order = np.argsort(bed.gid)
    np.testing.assert_array_equal(st["pos"], bed.x[order])
    np.testing.assert_array_equal(st["gid"], bed.gid[order])
    with pytest.raises(D.DemError) as e:
        gb.drive_wall(9, 1.0)
    assert e.value.status == D.DEM_ERR_INVALID
    with pytest.raises(D.DemError):
        gb.set_solver(dt=-1.0)
    gb.close()
    with pytest.raises(D.DemError) as e:
        D.Bed(bed.x, -bed.r, box=dict(lo=(0, 0, 0), hi=(1, 1, 1)))
    assert e.value.status == D.DEM_ERR_INVALID


# ------------------------------------------------------------------ full-size checks
def test_full_size_sampled_pair_set_and_invariants():
    """config 1 geometry as a jammed packing (~300k particles, bench launch configuration):
    sampled pair sets against the oracle's brute force, cones, momentum without walls/gravity."""
    bed = synth.banded_bed((0.4, 0.4, 0.3), [(0.0, 0.06, 2e-3), (0.06, 0.3, 4e-3)], 1001, spacing=2.0)
    D = dem()
    gb = D.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=dict(dt=5e-6, n_iter=20, gravity=(0, 0, 0)),
               box=dict(lo=bed.box_lo, hi=bed.box_hi, wall_mask=0))
    rho = 2600.0
    m = rho * np.pi * (2 * bed.r[np.argsort(bed.gid)]) ** 3 / 6
    p_before = (m[:, None] * gb.get_state()["vel"]).sum(0)
    gb.step(1)
    c = gb.get_contacts()
    st = gb.get_state()
    gb.close()
    # cones (fp32 impulses)
    inv = np.argsort(bed.gid)
    ka = (c["key"] >> np.uint64(32)).astype(np.int64)
    kb = (c["key"] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    Rs = bed.r[inv[ka]] * bed.r[inv[kb]] / (bed.r[inv[ka]] + bed.r[inv[kb]])
    Pn = c["P"][:, 0]
    assert (np.linalg.norm(c["P"][:, 1:4], axis=1) <= 0.4 * Pn * (1 + 1e-6) + 1e-30).all()
    assert (np.linalg.norm(c["P"][:, 4:7], axis=1) <= 0.1 * Rs * Pn * (1 + 1e-6) + 1e-30).all()
    # momentum: inter-particle impulses cancel
    p_after = (m[:, None] * st["vel"]).sum(0)
    scale = (m[:, None] * np.abs(st["vel"])).sum()
    assert np.abs(p_after - p_before).max() <= 1e-11 * scale
    # sampled pair sets vs brute force on the initial state
    rng = np.random.default_rng(5)
    sample = rng.choice(bed.n, 400, replace=False)
    Wo = oracle_world(bed, walls=False)
    ref = Wo.contacts_of(sample)
    sg = set(bed.gid[sample].tolist())
    mine = c[np.isin(ka, list(sg)) | np.isin(kb, list(sg))]
    np.testing.assert_array_equal(np.sort(mine["key"]), ref["key"])
    assert len(ref) > 1000


def test_force_limited_motor_vs_oracle():
    """Eq. 4 motor limits: a grouser plate pressed down by a velocity motor (-0.3 m/s)
    limited to 0.2 N, and sheared along x by a motor limited to 0.05 N; 60 steps on both sides:
    pair sets every step, plate positions, contact and motor forces."""
    bed = _small_bed_for_plates(47)
    lo = [(-0.006, -0.006, 0.0), (-0.006, -0.006, -0.003), (0.003, -0.006, -0.003)]
    hi = [(0.006, 0.006, 0.002), (-0.004, 0.006, 0.0), (0.005, 0.006, 0.0)]
    top = bed.x[:, 2].max() + 2.0e-3
    P = O.make_plate(lo, hi, pos=(0.015, 0.015, top), mass=0.02)
    P.mode[2], P.target[2], P.limit[2], P.fmin[2], P.fmax[2] = 1, -0.3, 1, -0.2, 0.2
    P.mode[0], P.target[0], P.limit[0], P.fmin[0], P.fmax[0] = 1, 0.1, 1, -0.05, 0.05
    Wo = oracle_world(bed, plates=[P])
    po = oracle_params(30, 1e-5)
    gb = gpu_bed(bed, dt=1e-5, n_iter=30)
    pid = gb.add_plate(lo, hi, (0.015, 0.015, top), 0.02)
    gb.drive_plate(pid, 2, 1, -0.3, 0.0, -0.2, 0.2)
    gb.drive_plate(pid, 0, 1, 0.1, 0.0, -0.05, 0.05)
    saturated = 0
    try:
        for s in range(60):
            c_ref, _, _ = Wo.step(po)
            gb.step(1)
            c = gb.get_contacts()
            assert np.array_equal(c["key"], c_ref["key"]), s
            g = gb.get_plate(pid)
            for k in (0, 2):
                assert g["pos"][k] == pytest.approx(Wo.plates[0].pos[k], abs=1e-12), (s, k)
                assert g["motor_force"][k] == pytest.approx(Wo.plates[0].motor[k], rel=1e-6, abs=1e-9), (s, k)
            saturated += g["motor_force"][2] == -0.2
    finally:
        gb.close()
    assert (c_ref["key"] & np.uint64(0xFFFFFFFF) >= np.uint64(O.PLATE_KEY_BASE)).sum() > 0
    assert saturated > 10
    with pytest.raises(Exception):
        gb2 = gpu_bed(bed, dt=1e-5, n_iter=30)
        try:
            p2 = gb2.add_plate(lo, hi, (0.015, 0.015, top), 0.02)
            gb2.drive_plate(p2, 0, 1, 0.1, 0.0, 1.0, -1.0)          # f_min > f_max: DEM_ERR_INVALID
        finally:
            gb2.close()


def test_step_report_residuals_vs_oracle():
    """Step report: the max normal complementarity residual and the max cone
    excess at the final velocities, against the oracle's on the same step (config 0s, 92 sweeps).
    The residual of an unconverged Jacobi iterate is a small difference of large terms (measured:
    1.3601e-6 vs 1.3586e-6), held to 2 %; the cone excess to the fp32 rounding of P."""
    bed, hist = config0s()
    Wo = oracle_world(bed)
    Wo.hist = hist
    Wo.step(oracle_params(92, 1e-5, v_imp=1e30))
    ro = Wo.last_report
    gb = gpu_bed(bed, dt=1e-5, n_iter=92, v_impact=1e30)
    try:
        gb.set_state(bed.x, bed.r, bed.v, bed.w, bed.gid, hist=hist)
        rep = gb.step(1)
        Pmax = float(np.abs(gb.get_contacts()["P"][:, 0]).max())
    finally:
        gb.close()
    print("residual gpu", rep["max_normal_residual"], "oracle", ro.max_normal_residual,
          "cone gpu", rep["max_cone_excess"], "oracle", ro.max_cone_excess)
    assert ro.max_normal_residual > 0
    assert rep["max_normal_residual"] == pytest.approx(ro.max_normal_residual, rel=0.02)
    assert 0.0 <= rep["max_cone_excess"] <= ro.max_cone_excess + 1e-6 * Pmax


def test_divergence_names_first_offending_contact_and_rolls_back():
    """S:365 / S:385: a NaN in the state makes the step fail atomically; the error names the
    step and the first offending contact (smallest key among contacts with non-finite impulses).
    One sweep, no impact stage: exactly the contacts of the poisoned particle go non-finite."""
    D = dem()
    bed = synth.random_cloud(300, (0, 0, 0), (0.04, 0.04, 0.04), 1.5e-3, 3e-3, 23, v_scale=0.01)
    c_ref, _ = oracle_world(bed).detect(oracle_params(1, 1e-5))
    ka = (c_ref["key"] >> np.uint64(32)).astype(np.int64)
    kb = (c_ref["key"] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    victim = int(np.bincount(ka, minlength=300)[:300].argmax())          # a particle with contacts
    mine = (ka == victim) | (kb == victim)
    expect = int(c_ref["key"][mine].min())
    v = bed.v.copy()
    v[np.flatnonzero(bed.gid == victim)[0], 0] = np.nan
    b = D.Bed(bed.x, bed.r, v, bed.w, bed.gid, box=dict(lo=(0, 0, 0), hi=(0.04, 0.04, 0.04)),
              solver=dict(dt=1e-5, n_iter=1, v_impact=1e30))
    try:
        st0 = b.get_state()
        with pytest.raises(D.DivergedError) as ei:
            b.step(1)
        st1 = b.get_state()
    finally:
        b.close()
    msg = str(ei.value)
    assert "step 1 diverged" in msg and f"contact key {expect} " in msg, (msg, expect)
    assert np.array_equal(st0["pos"], st1["pos"])                       # rolled back


def _big_sphere_bed():
    """One 12 mm sphere inside a shell of 1.5 mm spheres pressed onto it (overlapping slightly),
    plus a loose cloud: the big sphere's contact list has far more than 32 entries, so the
    packed sweep cuts it into 32-entry pieces (sweep_t2.cu long-list path)."""
    rng = np.random.default_rng(7)
    R, r = 0.012, 1.5e-3
    c = np.array([0.03, 0.03, 0.03])
    n = 140
    k = np.arange(n) + 0.5                                       # Fibonacci sphere directions
    phi = np.arccos(1 - 2 * k / n)
    th = np.pi * (1 + 5 ** 0.5) * k
    d = np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], axis=1)
    shell = c + (R + r - 2e-5) * d
    cloud = synth.random_cloud(200, (0.0, 0.0, 0.0), (0.06, 0.06, 0.06), 1.2e-3, 2e-3, 8)
    far = np.linalg.norm(cloud.x - c, axis=1) > R + 5e-3
    x = np.concatenate([c[None], shell, cloud.x[far]])
    rr = np.concatenate([[R], np.full(n, r), cloud.r[far]])
    v = rng.normal(0, 0.01, x.shape)
    b = synth.Bed(x=x, r=rr, v=v, w=np.zeros_like(x), gid=np.arange(len(rr), dtype=np.uint32),
                  box_lo=(0.0, 0.0, 0.0), box_hi=(0.06, 0.06, 0.06), name="big-sphere")
    return b


def test_long_contact_list_vs_oracle():
    bed = _big_sphere_bed()
    res = compare_step(bed, n_it=40, dt=1e-5, n_steps=2)
    assert res["pairs_equal"], res
    assert res["force_err"] <= TOL_F and res["torque_err"] <= TOL_F, res
    c_ref, _ = oracle_world(bed).detect(oracle_params(1, 1e-5))
    ka = (c_ref["key"] >> np.uint64(32)).astype(np.int64)
    kb = (c_ref["key"] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    assert int(((ka == 0) | (kb == 0)).sum()) > 100                    # > 3 chunks of 32


def test_monolithic_plate_momentum_and_oracle():
    """R18b: a free plate (all axes force-driven, F = 0) strikes a free sphere with gravity off:
    total momentum conserved at every step (the plate takes exactly the impulses the sphere
    gives, through the impact and main stages), and the trajectory matches the oracle's."""
    D = dem()
    r = 4.25e-3
    m_s = 2200.0 * 4.0 / 3.0 * np.pi * r ** 3
    x0 = np.array([[0.05 - 0.01 - r - 2e-5, 0.001, 0.048]])
    P = O.make_plate([(-0.01, -0.01, -0.01)], [(0.01, 0.01, 0.01)], pos=(0.05, 0.0, 0.05), mass=0.02)
    for k in range(3):
        P.mode[k], P.target[k] = 2, 0.0
    P.vel[0] = -0.3
    Wo = O.OracleWorld(x0, np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], plates=[P])
    po = O.make_params(h=1e-5, n_it=30, E=1e9, nu=0.15, rho=2200.0, g=(0, 0, 0), plate_coupling=1)
    b = D.Bed(x0, [r], box=dict(lo=(-1, -1, -1), hi=(1, 1, 1), wall_mask=0),
              material=dict(density=2200.0, youngs=1e9, poisson=0.15),
              solver=dict(dt=1e-5, n_iter=30, gravity=(0, 0, 0), plate_coupling=1))
    pid = b.add_plate([(-0.01, -0.01, -0.01)], [(0.01, 0.01, 0.01)], (0.05, 0.0, 0.05), 0.02)
    for k in range(3):
        b.drive_plate(pid, k, D.AXIS_FORCE, 0.0)
    # the plate starts at -0.3 m/s along x: one kinematic step sets that velocity on both sides
    b.drive_plate(pid, 0, D.AXIS_VELOCITY, -0.3)
    Wo.plates[0].mode[0], Wo.plates[0].target[0], Wo.plates[0].vel[0] = 1, -0.3, -0.3
    b.step(1)
    Wo.step(po)
    b.drive_plate(pid, 0, D.AXIS_FORCE, 0.0)
    Wo.plates[0].mode[0], Wo.plates[0].target[0] = 2, 0.0
    try:
        st = b.get_state()
        mom0 = 0.02 * np.array(b.get_plate(pid)["vel"]) + m_s * st["vel"][0]
        hit = 0
        for _ in range(80):
            rep = b.step(1)
            Wo.step(po)
            hit += rep["n_plate"]
            st = b.get_state()
            g = b.get_plate(pid)
            mom = 0.02 * np.array(g["vel"]) + m_s * st["vel"][0]
            assert np.abs(mom - mom0).max() <= 1e-9 * 0.02 * 0.3
            assert g["pos"][0] == pytest.approx(Wo.plates[0].pos[0], abs=1e-12)
            assert st["vel"][0][0] == pytest.approx(Wo.v[0, 0], rel=1e-5, abs=1e-9)
    finally:
        b.close()
    assert hit > 0 and st["vel"][0][0] < -0.05


@pytest.mark.slow
@pytest.mark.parametrize("wl,n_min,nc_min", [("config4-geom", 14_000_000, 30_000_000),
                                              ("config2-count", 2_000_000, 1_000_000)])
def test_full_size_bench_configuration_sampled(wl, n_min, nc_min):
    """A bench workload at full size (config4-geom: 14.6 M spheres in three bands; config2-count:
    2.1 M spheres on the Eq. 1 profile d 4 -> 32 mm, four grid levels), from the on-device
    generator, N_it from Eqs. 8 + 10, the shipped canonical packed sweep, walls and gravity off:
    sampled pair sets of 300 spheres against the oracle's brute force over the whole bed, cones at
    fp32 rounding (step report), total momentum conserved, and the step bit-reproducible run to
    run."""
    import bench
    D = dem()
    w = bench.WORKLOADS[wl]
    gen = bench.device_generator(wl)
    box = dict(lo=(0.0, 0.0, 0.0), hi=w["dims"], wall_mask=0)
    n_it = D.plan_iterations(bench.workload_network_length(w), 0.02)
    solver = dict(dt=w["dt"], n_iter=n_it, gravity=(0.0, 0.0, 0.0))

    def run():
        b = D.Bed(generator=gen, solver=solver, box=box)
        st0 = b.get_state()
        rep = b.step(1)
        st1 = b.get_state()
        c = b.get_contacts()
        b.close()
        return st0, rep, st1, c
    st0, rep, st1, c = run()
    n = len(st0["radius"])
    assert n > n_min and rep["n_contacts"] > nc_min
    # cones: the report's max excess is the fp32 rounding of P
    Pn_max = float(c["P"][:, 0].max())
    assert rep["max_cone_excess"] <= 1e-6 * Pn_max
    # momentum (inter-particle impulses cancel)
    m = 2600.0 * np.pi * (2 * st0["radius"]) ** 3 / 6
    p0 = (m[:, None] * st0["vel"]).sum(0)
    p1 = (m[:, None] * st1["vel"]).sum(0)
    assert np.abs(p1 - p0).max() <= 1e-9 * (m[:, None] * np.abs(st1["vel"])).sum()
    # sampled pair sets on the initial state, brute force over all 14.6 M spheres
    rng = np.random.default_rng(4)
    sample = rng.choice(n, 300, replace=False)
    Wo = O.OracleWorld(st0["pos"], st0["vel"], st0["angvel"], st0["radius"], st0["gid"])
    ref = Wo.contacts_of(sample)
    sg = set(st0["gid"][sample].tolist())
    ka = (c["key"] >> np.uint64(32)).astype(np.int64)
    kb = (c["key"] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    sel = np.isin(ka, list(sg)) | np.isin(kb, list(sg))
    np.testing.assert_array_equal(np.sort(c["key"][sel]), ref["key"])
    assert len(ref) > 500
    # run to run
    _, rep2, st2, _ = run()
    assert np.array_equal(st1["vel"], st2["vel"]) and rep2["n_contacts"] == rep["n_contacts"]


def test_checkpoint_resume_bit_identical(tmp_path):
    """checkpoint.save / load: a bed saved after 30 steps and resumed continues bit-identically
    to the uninterrupted run (state in fp64, the history's fp32 impulses round-trip exactly)."""
    from paper_2501_05300_b200 import checkpoint as CP
    D = dem()
    bed = synth.random_cloud(500, (0.002, 0.002, 0.002), (0.038, 0.038, 0.03), 1.5e-3, 3e-3, 12, v_scale=0.1)
    kw = dict(solver=dict(dt=2e-5, n_iter=30), box=dict(lo=(0, 0, 0), hi=(0.04, 0.04, 0.06)))
    a = D.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, **kw)
    a.step(30)
    p = str(tmp_path / "bed.npz")
    CP.save(a, p, meta=dict(note="test"))
    a.step(20)
    b = CP.load(p)
    b.step(20)
    try:
        sa, sb = a.get_state(), b.get_state()
        for k in ("pos", "vel", "angvel"):
            assert np.array_equal(sa[k], sb[k]), k
        assert np.array_equal(a.get_contacts()["P"], b.get_contacts()["P"])
        assert b.checkpoint_meta == {"note": "test"}
    finally:
        a.close()
        b.close()


def test_checkpoint_guards(tmp_path):
    """checkpoint.save before any step writes an empty history (the resumed bed steps like a
    fresh one); a moved or moving wall, or a plate, is refused (not captured)."""
    from paper_2501_05300_b200 import checkpoint as CP
    D = dem()
    bed = synth.random_cloud(300, (0.002, 0.002, 0.002), (0.038, 0.038, 0.03), 1.5e-3, 3e-3, 15, v_scale=0.1)
    kw = dict(solver=dict(dt=2e-5, n_iter=20), box=dict(lo=(0, 0, 0), hi=(0.04, 0.04, 0.06)))
    a = D.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, **kw)
    p = str(tmp_path / "fresh.npz")
    try:
        CP.save(a, p)
        b = CP.load(p)
        try:
            a.step(5)
            b.step(5)
            assert np.array_equal(a.get_state()["pos"], b.get_state()["pos"])
        finally:
            b.close()
        a.drive_wall(1, -0.01)
        with pytest.raises(ValueError):       # the wall is moving
            CP.save(a, p)
        a.step(1)
        a.drive_wall(1, 0.0)
        with pytest.raises(ValueError):       # the wall has moved
            CP.save(a, p)
    finally:
        a.close()


def test_add_and_remove_particles_match_recreate():
    """dem_add_particles / dem_remove_particles keep the state and the contact history: the run
    continues bit-identically to re-creating the bed from the edited state with the history
    handed back through dem_set_state."""
    D = dem()
    bed = synth.random_cloud(400, (0.002, 0.002, 0.002), (0.038, 0.038, 0.025), 1.5e-3, 3e-3, 13, v_scale=0.05)
    kw = dict(solver=dict(dt=2e-5, n_iter=30), box=dict(lo=(0, 0, 0), hi=(0.04, 0.04, 0.06)))
    extra = synth.random_cloud(60, (0.005, 0.005, 0.04), (0.035, 0.035, 0.05), 1.5e-3, 2.5e-3, 14)
    xg = (np.arange(60) + 1000).astype(np.uint32)
    a = D.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, **kw)
    a.step(15)
    st, c = a.get_state(), a.get_contacts()
    a.add_particles(extra.x, extra.r, gid=xg)
    a.step(10)
    removed = a.remove_particles(2, -1.0, 0.02)
    a.step(10)
    # the same through re-creation
    x = np.concatenate([st["pos"], extra.x]); r = np.concatenate([st["radius"], extra.r])
    v = np.concatenate([st["vel"], np.zeros((60, 3))]); w = np.concatenate([st["angvel"], np.zeros((60, 3))])
    g = np.concatenate([st["gid"], xg])
    b = D.Bed(x, r, v, w, g, **kw)
    b.set_state(x, r, v, w, g, hist=c)
    b.step(10)
    st2, c2 = b.get_state(), b.get_contacts()
    keep = st2["pos"][:, 2] <= 0.02
    b.close()
    b = D.Bed(st2["pos"][keep], st2["radius"][keep], st2["vel"][keep], st2["angvel"][keep], st2["gid"][keep], **kw)
    b.set_state(st2["pos"][keep], st2["radius"][keep], st2["vel"][keep], st2["angvel"][keep], st2["gid"][keep], hist=c2)
    b.step(10)
    try:
        assert removed == int((~keep).sum()) and removed > 0
        sa, sb = a.get_state(), b.get_state()
        for k in ("gid", "pos", "vel", "angvel"):
            assert np.array_equal(sa[k], sb[k]), k
    finally:
        a.close()
        b.close()


@pytest.mark.gpu
def test_add_particles_on_dense_bed_matches_recreate():
    """Regression: a particle reallocation must leave the candidate-sized key/sort scratch intact.
    On a jammed FCC bed the candidate count is several times N, so history export and the
    candidate sorts after dem_add_particles overran a scratch resized to 1.5 N."""
    D = dem()
    bed = synth.banded_bed((0.05, 0.05, 0.03), [(0.0, 0.03, 1.5e-3)], 21, spacing=2.0)
    kw = dict(solver=dict(dt=1e-5, n_iter=20), box=dict(lo=(0, 0, 0), hi=(0.05, 0.05, 0.06)))
    n_x = 40
    extra = synth.random_cloud(n_x, (0.006, 0.006, 0.04), (0.044, 0.044, 0.05), 1.2e-3, 1.5e-3, 22)
    xg = (np.arange(n_x) + bed.n + 100).astype(np.uint32)
    a = D.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, **kw)
    rep = a.step(3)
    assert rep["n_contacts"] > 2 * bed.n
    st, c = a.get_state(), a.get_contacts()
    a.add_particles(extra.x, extra.r, gid=xg)
    a.step(6)
    x = np.concatenate([st["pos"], extra.x]); r = np.concatenate([st["radius"], extra.r])
    v = np.concatenate([st["vel"], np.zeros((n_x, 3))]); w = np.concatenate([st["angvel"], np.zeros((n_x, 3))])
    g = np.concatenate([st["gid"], xg])
    b = D.Bed(x, r, v, w, g, **kw)
    b.set_state(x, r, v, w, g, hist=c)
    b.step(6)
    try:
        sa, sb = a.get_state(), b.get_state()
        for k in ("gid", "pos", "vel", "angvel"):
            assert np.array_equal(sa[k], sb[k]), k
        ca, cb = a.get_contacts(), b.get_contacts()
        assert np.array_equal(ca["key"], cb["key"]) and np.array_equal(ca["P"], cb["P"])
    finally:
        a.close()
        b.close()


@pytest.mark.gpu
def test_remove_all_then_add_matches_fresh_bed():
    """Edge cases of the particle-set edits: removing every particle leaves a valid empty bed that
    steps; particles added to it then evolve bit-identically to a fresh bed of the same particles."""
    D = dem()
    kw = dict(solver=dict(dt=2e-5, n_iter=25), box=dict(lo=(0, 0, 0), hi=(0.04, 0.04, 0.06)))
    b0 = synth.random_cloud(300, (0.003, 0.003, 0.003), (0.037, 0.037, 0.03), 1.5e-3, 3e-3, 31, v_scale=0.05)
    b1 = synth.random_cloud(200, (0.003, 0.003, 0.003), (0.037, 0.037, 0.03), 1.5e-3, 3e-3, 32, v_scale=0.05)
    a = D.Bed(b0.x, b0.r, b0.v, b0.w, b0.gid, **kw)
    f = D.Bed(b1.x, b1.r, b1.v, b1.w, b1.gid, **kw)
    try:
        a.step(5)
        assert a.remove_particles(2, 1.0, 2.0) == 300    # every centre lies outside [1, 2]
        assert a.get_state()["pos"].shape == (0, 3)
        a.step(2)                                   # an empty bed steps
        assert a.remove_particles(0, -1.0, 1.0) == 0     # nothing to remove from an empty bed
        a.add_particles(b1.x, b1.r, b1.v, b1.w, gid=b1.gid)
        a.step(8)
        f.step(8)
        sa, sf = a.get_state(), f.get_state()
        for k in ("gid", "pos", "vel", "angvel"):
            assert np.array_equal(sa[k], sf[k]), k
    finally:
        a.close()
        f.close()


@pytest.mark.slow
@pytest.mark.parametrize("n_it", [1, 3])
def test_full_size_sampled_sweep_outputs(n_it):
    """The sweep's OUTPUTS at the bench's full size (config4-geom, 14.6 M spheres, the bench's
    launch configuration), sampled: after one step of n_it Jacobi sweeps from the generator state
    (zero history, no gravity, no walls), a particle's velocity and spin depend only on the
    particles within n_it contact hops of it (the Jacobi iterate moves information one contact
    per sweep) and on the contact counts of those within n_it - 1 hops (mass splitting, C22).
    So the oracle computes each sampled particle's result one by one on the sub-bed of its
    n_it + 1 hop neighbourhood.  Bar: 1e-9 of the largest velocity / spin change
    (measured: 2.5e-11 at n_it = 1 on a 695-sphere sub-bed; 3.4e-11 / 4.1e-11 in velocity / spin at
    n_it = 3 on 3,856 spheres)."""
    import bench
    from scipy.spatial import cKDTree
    D = dem()
    wl = "config4-geom"
    w = bench.WORKLOADS[wl]
    box = dict(lo=(0.0, 0.0, 0.0), hi=w["dims"], wall_mask=0)
    b = D.Bed(generator=bench.device_generator(wl), solver=dict(dt=w["dt"], n_iter=n_it, gravity=(0.0, 0.0, 0.0)),
              box=box)
    try:
        st0 = b.get_state()
        rep = b.step(1)
        st1 = b.get_state()
    finally:
        b.close()
    assert rep["impact_fired"] == 0 and rep["n_contacts"] > 30_000_000
    x, r = st0["pos"], st0["radius"]
    tree = cKDTree(x)
    rmax = float(r.max())
    rng = np.random.default_rng(11)
    sample = rng.choice(len(r), 24, replace=False)

    def touching(idx):
        out = set()
        for i, nb in zip(idx, tree.query_ball_point(x[idx], r[idx] + rmax)):
            nb = np.asarray(nb)
            d = np.linalg.norm(x[nb] - x[i], axis=1)
            out.update(nb[(d < r[nb] + r[i]) & (nb != i)].tolist())
        return out

    local, front = set(sample.tolist()), list(sample.tolist())
    for _ in range(n_it + 1):
        nxt = touching(np.asarray(front)) - local
        local |= nxt
        front = sorted(nxt)
    loc = np.array(sorted(local))
    Wo = O.OracleWorld(x[loc], st0["vel"][loc], st0["angvel"][loc], r[loc], st0["gid"][loc])
    Wo.step(oracle_params(n_it, w["dt"], g=(0.0, 0.0, 0.0)))
    pos_in = np.searchsorted(loc, sample)
    dv_ref = Wo.v[pos_in] - st0["vel"][sample]
    dw_ref = Wo.w[pos_in] - st0["angvel"][sample]
    dv = st1["vel"][sample] - st0["vel"][sample]
    dw = st1["angvel"][sample] - st0["angvel"][sample]
    sv, sw = np.abs(dv_ref).max(), np.abs(dw_ref).max()
    print("n_it", n_it, "sub-bed", len(loc), "max |dv|", sv, "err", np.abs(dv - dv_ref).max(), "max |dw|", sw,
          "err", np.abs(dw - dw_ref).max())
    assert sv > 1e-3
    assert np.abs(dv - dv_ref).max() <= 1e-9 * sv
    # spin scale floor |dv| / r (the first sweep turns nothing: no tangential relative velocity yet)
    assert np.abs(dw - dw_ref).max() <= 1e-9 * max(sw, sv / float(np.median(r)))
