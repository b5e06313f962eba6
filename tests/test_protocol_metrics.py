"""Plate protocol metrics and normalised errors (PAPER §4.1-4.3; SPEC
extract_metrics / normalized_errors S:478-543), pinned to the paper's own numbers and to
constructed signals, plus the phase logic of run_plate_test driven through a stand-in bed."""
import numpy as np
import pytest

from paper_2501_05300_b200 import protocol as PR

AXIS_LOCKED, AXIS_VELOCITY, AXIS_FORCE = 0, 1, 2


def test_paper_low_gamma_aggregate_is_3p4_percent():
    # P:333 "starting at 3.4% in the low range"; component deviations from §4.1-4.2:
    # dz_static = 0.22 mm, dz_dyn = 4.4 mm, dcoef_peak = 0.004, dcoef_avg = 0.0237,
    # h_grouser = 43.0 mm, F_N,max = 2550 N
    ref = dict(static_sinkage=1.26e-3, dynamic_sinkage=70.8e-3, peak_traction=0.268, avg_traction=0.320)
    m = dict(static_sinkage=ref["static_sinkage"] + 0.22e-3, dynamic_sinkage=ref["dynamic_sinkage"] + 4.4e-3,
             peak_traction=ref["peak_traction"] + 0.004, avg_traction=ref["avg_traction"] + 0.0237)
    e = PR.normalized_errors(m, ref, 43.0e-3, 2550.0)
    assert round(100 * e["static_sinkage"], 2) == 0.51
    assert round(100 * e["dynamic_sinkage"], 1) == 10.2
    assert round(100 * e["peak_traction"], 2) == 0.40
    assert round(100 * e["avg_traction"], 2) == 2.37
    assert round(100 * e["aggregate"], 1) == 3.4


def test_normalized_errors_special_cases():
    ref = dict(static_sinkage=1e-3, dynamic_sinkage=0.07, peak_traction=0.27, avg_traction=0.32)
    e = PR.normalized_errors(ref, ref, 0.043, 2550.0)
    assert all(v == 0.0 for v in e.values())
    m = dict(ref, dynamic_sinkage=ref["dynamic_sinkage"] - 0.043)        # SPEC S:542 derived example
    e = PR.normalized_errors(m, ref, 0.043, 2550.0)
    assert e["dynamic_sinkage"] == pytest.approx(-1.0, abs=1e-12)
    assert e["aggregate"] == pytest.approx(0.25, abs=1e-12)
    # traction errors are force differences: a run at half the maximum load halves them
    m = dict(ref, avg_traction=ref["avg_traction"] + 0.1)
    assert PR.normalized_errors(m, ref, 0.043, 2550.0, F_N=1275.0)["avg_traction"] == pytest.approx(0.05)


def series(fn_s, fn_tr, dt=1e-4, proto=None):
    proto = proto or PR.PlateProtocol(F_N=2550.0)
    t = dt * np.arange(1, int(round(proto.t_end / dt)) + 1)
    return dict(t=t, sinkage=fn_s(t), traction=fn_tr(t)), proto


def test_constant_series_reproduce_constants():
    sr, proto = series(lambda t: np.full_like(t, 5e-3), lambda t: np.full_like(t, 0.3))
    m = PR.extract_metrics(sr, proto)
    assert m["static_sinkage"] == pytest.approx(5e-3, rel=1e-12)
    assert m["dynamic_sinkage"] == pytest.approx(5e-3, rel=1e-12)
    assert m["peak_traction"] == pytest.approx(0.3, rel=1e-12)
    assert m["avg_traction"] == pytest.approx(0.3, rel=1e-12)
    assert m["dynamic_sinkage_growth"] == pytest.approx(0.0, abs=1e-15)


def test_triangular_traction_peak():
    # traction peaking 0.4 at t = 2.75 s.  The 25 ms centred average of a symmetric
    # triangle of slope k at its apex is 0.4 - k w / 4 (mean of the tent over [-w/2, w/2]; the
    # sampled mean differs from it by less than k dt).
    k = 0.4
    sr, proto = series(lambda t: 1e-3 * t, lambda t: np.maximum(0.0, 0.4 - k * np.abs(t - 2.75)))
    m = PR.extract_metrics(sr, proto)
    assert m["peak_traction"] == pytest.approx(0.4 - k * proto.smooth / 4, abs=k * 1e-4)
    # a tent narrower than nothing: smoothing off reproduces the apex exactly
    proto0 = PR.PlateProtocol(F_N=1.0, smooth=0.0)
    assert PR.extract_metrics(sr, proto0)["peak_traction"] == pytest.approx(0.4, abs=1e-12)
    # linear sinkage: window means are the window midpoints
    assert m["static_sinkage"] == pytest.approx(1e-3 * (proto.t_I_end - proto.window / 2), rel=1e-3)
    assert m["dynamic_sinkage"] == pytest.approx(1e-3 * (proto.t_end - proto.window / 2), rel=1e-3)


def test_metrics_invariant_under_2x_resampling():
    f_s = lambda t: 1e-3 * (1 - np.exp(-t)) + 2e-3 * np.sin(3 * t) ** 2
    f_tr = lambda t: 0.3 + 0.05 * np.sin(7 * t) * np.exp(-(t - 2.6) ** 2)
    a, proto = series(f_s, f_tr, dt=2e-4)
    b, _ = series(f_s, f_tr, dt=1e-4)
    ma, mb = PR.extract_metrics(a, proto), PR.extract_metrics(b, proto)
    for k in ma:
        assert ma[k] == pytest.approx(mb[k], rel=2e-3, abs=1e-6), k


def test_short_series_rejected():
    sr, proto = series(lambda t: 0 * t, lambda t: 0 * t)
    cut = {k: v[: len(v) // 2] for k, v in sr.items()}
    with pytest.raises(ValueError):
        PR.extract_metrics(cut, proto)


def test_surface_datum_on_lattice():
    # square columns of 1 mm spheres, stacks of different heights: datum = mean column top
    r = 0.5e-3
    pos, rad, tops = [], [], []
    for i in range(4):
        for j in range(4):
            h = 3 + (i + j) % 3
            for k in range(h):
                pos.append(((i + 0.5) * 2 * r, (j + 0.5) * 2 * r, r + 2 * r * k))
                rad.append(r)
            tops.append(2 * r * h)
    d = PR.surface_datum(np.array(pos), np.array(rad), (4 * r, 4 * r), (4 * r, 4 * r))
    assert d == pytest.approx(np.mean(tops), rel=1e-12)


class StandInBed:
    """Duck-typed bed: a plate whose contact reaction is a fixed function of time; records the
    drive commands run_plate_test issues (host logic of the protocol only)."""

    def __init__(self, dt, contact=lambda t: 1):
        self.dt, self.t, self.cmds, self.contact = dt, 0.0, [], contact
        self.z, self.x, self.mode = 0.0, 0.0, {}

    def drive_plate(self, plate, axis, mode, target, ramp_time=0.0, f_min=-np.inf, f_max=np.inf):
        self.cmds.append((round(self.t / self.dt), axis, mode, target, ramp_time))
        self.mode[axis] = (mode, target, ramp_time, self.t)

    def step(self, n=1):
        self.t += self.dt
        m, u, ramp, t0 = self.mode.get(0, (AXIS_LOCKED, 0, 0, 0))
        if m == AXIS_VELOCITY:
            self.x += self.dt * u * min(1.0, (self.t - self.dt - t0) / ramp if ramp else 1.0)
        self.z -= 1e-6
        return {"time": self.t}

    def get_plate(self, plate):
        F = -self.mode[2][1]
        return {"pos": [self.x, 0.0, self.z], "vel": [0, 0, 0], "force": [-0.3 * F, 0.0, F],
                "motor_force": [0.3 * F, 0.0, -F], "n_contacts": self.contact(self.t)}


def test_run_plate_test_phase_logic():
    proto = PR.PlateProtocol(F_N=10.0, t_ramp=0.01, t_I_end=0.02, u_shear=0.1, t_shear_ramp=0.005,
                             t_II_end=0.025, t_end=0.04, window=0.005, smooth=0.001)
    dt = 1e-4
    bed = StandInBed(dt)
    sr = PR.run_plate_test(bed, 0, proto, dt, z_datum=0.0)
    assert len(sr["t"]) == 400
    force_cmds = [c for c in bed.cmds if c[1] == 2]
    assert all(c[2] == AXIS_FORCE for c in force_cmds)
    # phase I: linear ramp of the load to F_N over t_ramp, then held
    f = np.array([-c[3] for c in force_cmds[:200]])
    assert np.allclose(f[:100], 10.0 * np.arange(1, 101) * dt / 0.01)
    assert np.all(f[100:] == 10.0)
    # the horizontal axis is locked in phase I and switched to the velocity ramp at t_I_end
    shear = [c for c in bed.cmds if c[1] == 0]
    assert shear[0][2] == AXIS_LOCKED and shear[-1] == (200, 0, AXIS_VELOCITY, 0.1, 0.005)
    assert len(bed.cmds) == 1 + 200 + 1 + 1
    assert np.allclose(sr["traction"][150:], 0.3)
    m = PR.extract_metrics(sr, proto)
    assert m["avg_traction"] == pytest.approx(0.3)
    assert m["dynamic_sinkage"] > m["static_sinkage"] > 0


def test_run_plate_test_faults():
    proto = PR.PlateProtocol(F_N=10.0, t_ramp=0.01, t_I_end=0.02, t_II_end=0.025, t_end=0.4, window=0.005,
                             smooth=0.001)
    with pytest.raises(PR.ExperimentFault):                       # F_N = 0
        PR.run_plate_test(StandInBed(1e-3), 0, PR.PlateProtocol(F_N=0.0), 1e-3, 0.0)
    lose = StandInBed(1e-3, contact=lambda t: 0 if t > 0.1 else 3)
    with pytest.raises(PR.ExperimentFault):                       # contact lost > 0.2 s
        PR.run_plate_test(lose, 0, proto, 1e-3, 0.0)
    brief = StandInBed(1e-3, contact=lambda t: 0 if 0.1 < t < 0.25 else 3)
    PR.run_plate_test(brief, 0, proto, 1e-3, 0.0)                  # a 0.15 s gap is tolerated


def test_write_csv(tmp_path):
    sr = {"t": np.array([1e-4, 2e-4]), "sinkage": np.array([0.0, 1e-6])}
    p = tmp_path / "run.csv"
    PR.write_csv(p, sr)
    rows = p.read_text().splitlines()
    assert rows[0] == "t,sinkage" and len(rows) == 3
    assert float(rows[2].split(",")[1]) == 1e-6
