"""Box-shaped consolidated drained triaxial test and Mohr-Coulomb fit (PAPER §3.2
P:166-202, Table 1; SPEC run_triaxial / mohr_coulomb_fit S:448-466).  Host-side orchestration of
the library's kinematic walls (dem_drive_wall) and wall reactions (dem_get_wall); every step of
the simulation runs in libdem.so.

Protocol (servo law, tolerances and windows: SPEC design decisions S:496-499):
  1. consolidation -- the four side walls and the top wall are servo-driven, inward normal
     velocity v = clamp(K (sigma_3 - sigma_wall), +-v_max), until every servo wall carries sigma_3
     within 2 % and holds it for `hold` seconds (fault after t_consolidate_max);
  2. shear -- the top wall moves down at the axial rate (5 mm/s) while the side walls keep
     sigma_2 = sigma_3 by the same servo; sigma_1 = the top wall's stress; stop at max_strain.
     Fault: a side-wall stress error above 5 % for longer than 0.5 s.
Peak deviatoric stress: max of the `smooth`-window centred moving average of sigma_1 - sigma_3.
Wall w = 2 axis + side (0 -x, 1 +x, 2 -y, 3 +y, 4 -z bottom, 5 +z top); the bottom is fixed.
Walls are frictionless, the box's own wall friction settings (zero by default).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SIDES = (0, 1, 2, 3)
TOP, BOTTOM = 5, 4


class ExperimentFault(RuntimeError):
    """The servo could not establish or hold the confining stress."""


@dataclass
class TriaxialConfig:
    sigma3: float                    # confining stress sigma_2 = sigma_3 [Pa] (5, 15, 25 kPa)
    axial_rate: float = 5e-3         # top-wall speed [m/s]
    max_strain: float = 0.15         # axial strain at which the test stops (SPEC open question)
    K: float = 1e-6                  # servo gain [m/(s Pa)]
    v_max: float = 0.05              # servo speed clamp [m/s]
    tol: float = 0.02                # consolidation: every servo wall within 2 % of sigma_3
    hold: float = 0.05               # ... for this long [s]
    t_consolidate_max: float = 1.0   # consolidation budget [s] (SPEC open question: 1 s)
    fault_err: float = 0.05          # shear: side-wall stress error ...
    fault_time: float = 0.5          # ... tolerated for this long [s]
    smooth: float = 0.05             # peak detection window [s]


def box_and_stresses(bed):
    """Current box edge lengths (from the wall planes) and each wall's normal stress
    sigma_w = -F_w . n_w / A_w (compression positive)."""
    W = [bed.get_wall(w) for w in range(6)]
    L = [W[2 * a + 1]["point"][a] - W[2 * a]["point"][a] for a in range(3)]
    sig = []
    for w in range(6):
        a = w // 2
        area = L[(a + 1) % 3] * L[(a + 2) % 3]
        sig.append(-float(np.dot(W[w]["force"], W[w]["normal"])) / area)
    return L, sig


def servo(bed, walls, sig, target, cfg):
    for w in walls:
        v = cfg.K * (target - sig[w])
        bed.drive_wall(w, max(-cfg.v_max, min(cfg.v_max, v)))


def run_triaxial(bed, cfg: TriaxialConfig, dt: float, record_every: int = 1):
    """Runs consolidation and shear on `bed` (a dem.Bed in a box with all six walls); returns
    the shear-stage series (dict of arrays: t, strain, sigma1, sigma2 (x walls), sigma3 (y walls),
    sigma_dev = sigma1 - sigma_3 target) and the consolidation time."""
    if not cfg.sigma3 > 0 or not cfg.axial_rate > 0:
        raise ValueError("sigma3 and axial_rate must be positive")
    servo_walls = SIDES + (TOP,)
    t, ok_since = 0.0, None
    L, sig = box_and_stresses(bed)
    while True:
        servo(bed, servo_walls, sig, cfg.sigma3, cfg)
        bed.step(1)
        t += dt
        L, sig = box_and_stresses(bed)
        err = max(abs(sig[w] - cfg.sigma3) for w in servo_walls) / cfg.sigma3
        if err <= cfg.tol:
            ok_since = t if ok_since is None else ok_since
            if t - ok_since >= cfg.hold - 1e-12:
                break
        else:
            ok_since = None
        if t > cfg.t_consolidate_max:
            raise ExperimentFault(f"consolidation did not reach sigma3 within {cfg.tol:.0%} in "
                                  f"{cfg.t_consolidate_max} s (error {err:.3f})")
    t_cons = t
    H0 = L[2]
    cols = {k: [] for k in ("t", "strain", "sigma1", "sigma2", "sigma3", "sigma_dev", "height")}
    bed.drive_wall(TOP, cfg.axial_rate)
    bad, s = 0.0, 0
    while True:
        servo(bed, SIDES, sig, cfg.sigma3, cfg)
        bed.step(1)
        t += dt
        s += 1
        L, sig = box_and_stresses(bed)
        strain = (H0 - L[2]) / H0
        lat = max(abs(sig[w] - cfg.sigma3) for w in SIDES) / cfg.sigma3
        bad = bad + dt if lat > cfg.fault_err else 0.0
        if bad > cfg.fault_time:
            raise ExperimentFault(f"side walls lost sigma3 (error {lat:.3f}) at strain {strain:.4f}")
        if s % record_every == 0:
            cols["t"].append(t - t_cons)
            cols["strain"].append(strain)
            cols["sigma1"].append(sig[TOP])
            cols["sigma2"].append(0.5 * (sig[0] + sig[1]))
            cols["sigma3"].append(0.5 * (sig[2] + sig[3]))
            cols["sigma_dev"].append(sig[TOP] - cfg.sigma3)
            cols["height"].append(L[2])
        if strain >= cfg.max_strain:
            break
    bed.drive_wall(TOP, 0.0)
    for w in SIDES:
        bed.drive_wall(w, 0.0)
    out = {k: np.asarray(v, float) for k, v in cols.items()}
    out["t_consolidation"] = t_cons
    return out


def peak_deviator(series, cfg: TriaxialConfig):
    """Peak of the centred moving average (window cfg.smooth, in time) of sigma_1 - sigma_3."""
    t, y = np.asarray(series["t"], float), np.asarray(series["sigma_dev"], float)
    if len(t) == 0:
        raise ValueError("empty series")
    c = np.concatenate(([0.0], np.cumsum(y)))
    lo = np.searchsorted(t, t - 0.5 * cfg.smooth, side="left")
    hi = np.searchsorted(t, t + 0.5 * cfg.smooth, side="right")
    return float(((c[hi] - c[lo]) / (hi - lo)).max())


def mohr_coulomb_fit(peaks):
    """PAPER P:180 / SPEC S:460: least-squares line q = a + b p through the peak Mohr circles'
    (p, q) = ((sigma1 + sigma3)/2, (sigma1 - sigma3)/2); sin(phi) = b, c = a / cos(phi).
    peaks: [(sigma3, sigma1_peak), ...]; returns (phi in degrees, c in Pa)."""
    pk = np.asarray(peaks, float).reshape(-1, 2)
    if len(np.unique(pk[:, 0])) < 2:
        raise ValueError("the fit needs at least two distinct confinements (singular otherwise)")
    p = 0.5 * (pk[:, 1] + pk[:, 0])
    q = 0.5 * (pk[:, 1] - pk[:, 0])
    A = np.stack([np.ones_like(p), p], axis=1)
    (a, b), *_ = np.linalg.lstsq(A, q, rcond=None)
    if not -1.0 < b < 1.0:
        raise ValueError(f"slope {b} is not a sine of a friction angle")
    phi = math.asin(b)
    return math.degrees(phi), a / math.cos(phi)
