"""Plate protocol (phases I-III, SPEC run_plate_test S:468-477) on the GPU: the
SPEC invariants of the recorded series and the four metrics against the same protocol run by
the oracle, on the refined mini bed of tests/golden/plate_mini_state.npz with a compressed
timeline (load 5 N ramped over 4 ms, held to 12 ms; pull 0.05 m/s ramped over 4 ms; end 40 ms).
"""
import numpy as np
import pytest

import oracle as O
from paper_2501_05300_b200 import protocol as PR
from tests.parity import gpu_bed, oracle_params, oracle_world
from tests.test_gpu_curves import mini_bed

pytestmark = [pytest.mark.gpu, pytest.mark.slow, pytest.mark.usefixtures("oracle_binning")]

DT, N_IT = 2e-5, 40
LO, HI = [(-0.01, -0.01, 0.0)], [(0.01, 0.01, 0.004)]
MASS = 0.05
PROTO = PR.PlateProtocol(F_N=5.0, t_ramp=4e-3, t_I_end=12e-3, u_shear=0.05, t_shear_ramp=4e-3, t_II_end=20e-3,
                         t_end=40e-3, window=4e-3, smooth=1e-3, max_contact_loss=2e-3)
PLATE_KEY_BASE, WALL_KEY_BASE = 0xFFFFF000, 0xFFFFFFF0


class OracleBed:
    """The oracle world behind the bed interface run_plate_test drives (drive semantics of
    dem_drive_plate, include/dem.h: a velocity ramp starts from rest at the call time)."""

    def __init__(self, bed, hist, pos):
        self.P = O.make_plate(LO, HI, pos=pos, mass=MASS)
        self.W = oracle_world(bed, plates=[self.P])
        self.W.hist = hist
        self.params = oracle_params(N_IT, DT)

    def drive_plate(self, plate, axis, mode, target, ramp_time=0.0, f_min=-np.inf, f_max=np.inf):
        P = self.W.plates[plate]
        P.mode[axis], P.target[axis], P.ramp[axis], P.t0[axis] = mode, target, ramp_time, self.W.time
        P.limit[axis] = int(mode == 1 and (f_min > -np.inf or f_max < np.inf))
        P.fmin[axis], P.fmax[axis] = f_min, f_max
        if mode == 0:
            P.vel[axis] = 0.0
        elif mode == 1 and not P.limit[axis]:
            P.vel[axis] = 0.0 if ramp_time > 0 else target

    def step(self, n=1):
        self.W.step(self.params, n)
        return {"time": self.W.time}

    def get_plate(self, plate):
        P = self.W.plates[plate]
        lo = (self.W.hist["key"] & np.uint64(0xFFFFFFFF)).astype(np.int64)
        base = PLATE_KEY_BASE + 16 * plate
        n = int(np.count_nonzero((lo >= base) & (lo < base + 16)))
        return {"pos": list(P.pos), "vel": list(P.vel), "force": list(P.force), "motor_force": list(P.motor),
                "n_contacts": n}


@pytest.fixture(scope="module")
def runs(oracle_binning):
    bed, hist = mini_bed()
    top = float((bed.x[:, 2] + bed.r).max())
    pos = (0.02, 0.02, top + 2e-4)
    datum = PR.surface_datum(bed.x, bed.r, pos[:2], (0.01, 0.01)) - LO[0][2]
    gb = gpu_bed(bed, dt=DT, n_iter=N_IT)
    gb.set_state(bed.x, bed.r, bed.v, bed.w, bed.gid, hist=hist)
    pid = gb.add_plate(LO, HI, pos, MASS)
    try:
        s_gpu = PR.run_plate_test(gb, pid, PROTO, DT, datum)
    finally:
        gb.close()
    s_ref = PR.run_plate_test(OracleBed(bed, hist, pos), 0, PROTO, DT, datum)
    return s_gpu, s_ref


def test_plate_x_follows_the_commanded_ramp(runs):
    # horizontal position in II/III = integral of the ramp within dt * u
    s, _ = runs
    t = s["t"]
    sh = t > PROTO.t_I_end + 1e-12
    x0 = s["plate_x"][~sh][-1]
    tau = t[sh] - PROTO.t_I_end
    r = PROTO.t_shear_ramp
    integral = PROTO.u_shear * np.where(tau < r, tau ** 2 / (2 * r), tau - r / 2)
    assert np.abs(s["plate_x"][sh] - x0 - integral).max() <= DT * PROTO.u_shear * (1 + 1e-9)


def test_force_axis_balance(runs):
    # force balance of a force-driven axis: m dv/dt = F_contact - F_N, so over any
    # window the mean measured normal force is F_N + m dv/T exactly (the staggered update).  The
    # SPEC's "within 2% of F_N over any 0.25 s window of phase III" is a steady-state statement at
    # full scale; on this 20 ms compressed phase III the plate still accelerates into the bed
    # (measured: mean 4.77 N of 5 N, all of it the plate's momentum change), so only a 10% bound.
    s, _ = runs
    t, z = s["t"], -s["sinkage"]
    v = np.diff(z) / DT                       # velocity used in the step ending at t[i + 1]
    w = t > PROTO.t_II_end
    i0, i1 = np.flatnonzero(w)[0], len(t) - 1
    lhs = s["F_N_measured"][i0:i1].mean()
    rhs = PROTO.F_N + MASS * (v[i1 - 1] - v[i0 - 1]) / ((i1 - i0) * DT)
    assert lhs == pytest.approx(rhs, rel=1e-6)
    assert abs(lhs - PROTO.F_N) <= 0.10 * PROTO.F_N, lhs


def test_metrics_match_oracle(runs):
    s_gpu, s_ref = runs
    m_gpu, m_ref = PR.extract_metrics(s_gpu, PROTO), PR.extract_metrics(s_ref, PROTO)
    print("gpu", m_gpu)
    print("oracle", m_ref)
    assert m_ref["static_sinkage"] > 0 and m_ref["dynamic_sinkage"] > m_ref["static_sinkage"]
    assert 0.05 < m_ref["avg_traction"] < 1.5
    # P:322-331 normalisation at this scale: grouser depth 4 mm, F_N,max = the load
    e = PR.normalized_errors(m_gpu, m_ref, 4e-3, PROTO.F_N)
    print("normalised errors", e)
    assert e["aggregate"] <= 0.02
    assert all(abs(e[k]) <= 0.04 for k in ("static_sinkage", "dynamic_sinkage", "peak_traction", "avg_traction"))
