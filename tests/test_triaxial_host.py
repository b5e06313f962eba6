"""Triaxial protocol host logic and the Mohr-Coulomb fit (PAPER §3.2 P:166-202;
SPEC S:448-466): the fit pinned to closed forms and the SPEC examples, the servo/shear
orchestration against a stand-in bed whose walls are linear springs."""
import math

import numpy as np
import pytest

from paper_2501_05300_b200 import triaxial as TX


def test_mohr_coulomb_cohesionless_30_degrees():
    # sigma1 = 3 sigma3 is exactly sin(phi) = 1/2
    phi, c = TX.mohr_coulomb_fit([(5e3, 15e3), (15e3, 45e3), (25e3, 75e3)])
    assert phi == pytest.approx(30.0, abs=1e-9)
    assert abs(c) < 1e-6


def test_mohr_coulomb_cohesion_intercept():
    # points on q = 0.5 p + c cos(phi) with c = 1000 Pa, phi = 30 deg
    p = np.array([10e3, 20e3, 35e3])
    q = 0.5 * p + 1000.0 * math.cos(math.radians(30.0))
    pk = [(pi - qi, pi + qi) for pi, qi in zip(p, q)]           # sigma3 = p - q, sigma1 = p + q
    phi, c = TX.mohr_coulomb_fit(pk)
    assert phi == pytest.approx(30.0, abs=1e-9) and c == pytest.approx(1000.0, rel=1e-9)


@pytest.mark.parametrize("phi_deg", [10.0, 34.3, 34.9, 33.2])
def test_mohr_coulomb_closed_form_failure_line(phi_deg):
    # cohesionless Mohr-Coulomb failure: sigma1 = sigma3 (1 + sin phi) / (1 - sin phi)
    # (Table 1 angles)
    s = math.sin(math.radians(phi_deg))
    pk = [(s3, s3 * (1 + s) / (1 - s)) for s3 in (5e3, 15e3, 25e3)]
    phi, c = TX.mohr_coulomb_fit(pk)
    assert phi == pytest.approx(phi_deg, abs=1e-9) and abs(c) < 1e-6


def test_mohr_coulomb_duplication_invariant_and_singular():
    pk = [(5e3, 16e3), (15e3, 44e3), (25e3, 77e3)]
    assert TX.mohr_coulomb_fit(pk + pk) == pytest.approx(TX.mohr_coulomb_fit(pk))
    with pytest.raises(ValueError):
        TX.mohr_coulomb_fit([(5e3, 15e3), (5e3, 16e3)])


def test_peak_deviator_smoothing():
    cfg = TX.TriaxialConfig(sigma3=1e3, smooth=0.05)
    t = 1e-4 * np.arange(1, 20001)
    y = 1e3 * np.maximum(0.0, 1.0 - np.abs(t - 1.0))                # tent of slope 1e3 Pa/s
    pk = TX.peak_deviator(dict(t=t, sigma_dev=y), cfg)
    assert pk == pytest.approx(1e3 - 1e3 * cfg.smooth / 4, abs=1e3 * 1e-4)


class SpringBox:
    """Stand-in bed: a box whose walls move with their commanded inward velocities and carry a
    stress k * (L0 - L) along each axis (a linear elastic sample)."""

    def __init__(self, L0=(0.05, 0.05, 0.05), k=4e6, L_start=None):
        self.L0 = np.array(L0, float)
        self.lo = np.zeros(3)
        self.hi = np.array(L_start if L_start is not None else L0, float)
        self.v = np.zeros(6)
        self.k, self.dt = k, 1e-4

    def drive_wall(self, w, v):
        self.v[w] = v

    def step(self, n=1):
        for _ in range(n):
            for w in range(6):
                a = w // 2
                if w % 2 == 0:
                    self.lo[a] += self.dt * self.v[w]
                else:
                    self.hi[a] -= self.dt * self.v[w]
        return {}

    def get_wall(self, w):
        a = w // 2
        L = self.hi - self.lo
        sig = self.k * max(0.0, self.L0[a] - L[a])
        area = L[(a + 1) % 3] * L[(a + 2) % 3]
        n = np.zeros(3)
        n[a] = 1.0 if w % 2 == 0 else -1.0
        point = self.lo.copy() if w % 2 == 0 else self.hi.copy()
        return {"point": list(point), "normal": list(n), "velocity": self.v[w], "force": list(-sig * area * n),
                "n_contacts": 1}


def test_servo_consolidation_and_shear_on_springs():
    cfg = TX.TriaxialConfig(sigma3=5e3, axial_rate=5e-3, max_strain=0.02, hold=0.02)
    box = SpringBox()
    out = TX.run_triaxial(box, cfg, dt=box.dt)
    # consolidation reached: side strain 5e3 / 4e6 = 1.25e-3 per axis
    assert out["t_consolidation"] < cfg.t_consolidate_max
    assert np.abs(out["sigma3"] / cfg.sigma3 - 1).max() < cfg.fault_err
    # shear: the top wall moved at the axial rate; sigma1 = k (L0 - H) grows linearly with it
    H = out["height"]
    assert np.allclose(np.diff(H), -cfg.axial_rate * box.dt, rtol=1e-9, atol=1e-15)
    assert np.allclose(out["sigma1"], box.k * (box.L0[2] - H), rtol=1e-9)
    assert out["strain"][-1] >= cfg.max_strain
    assert abs(out["sigma_dev"][0]) <= 1.01 * cfg.tol * cfg.sigma3      # consolidated: sigma1 = sigma3 (2 %)
    assert out["sigma_dev"][-1] > 10 * cfg.tol * cfg.sigma3


def test_consolidation_fault():
    cfg = TX.TriaxialConfig(sigma3=5e3, t_consolidate_max=0.05, v_max=1e-4)   # far too slow a servo
    with pytest.raises(TX.ExperimentFault):
        TX.run_triaxial(SpringBox(L_start=(0.06, 0.06, 0.06)), cfg, dt=1e-4)
