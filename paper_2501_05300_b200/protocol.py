"""Plate pressure-sinkage and shear-displacement protocol and its metrics (PAPER
§3.3, §4.1-4.3; SPEC run_plate_test / extract_metrics / normalized_errors
S:468-543).  Host-side orchestration of the library's plate drives and the arithmetic on the
recorded series; every step of the simulation runs in libdem.so.

Phases: I -- the vertical axis is force-driven, the load ramps linearly from
0 to F_N over t_ramp and holds (horizontal axis locked) until t_I_end; II/III -- the horizontal
axis is velocity-driven, its speed ramped from 0 to u over t_shear_ramp ("increased
linearly from 0 to 100 mm/s over 0.1 s") then constant until t_end, the vertical axis still at
F_N.  Recorded per step: t, sinkage (datum: the surface under the plate at t = 0), the applied
load, the measured normal contact force, the pull force F_T (the horizontal motor's constraint
force lambda of Eq. 4, which at constant speed is minus the horizontal contact reaction) and
the traction F_T / F_N.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import dem as D


@dataclass
class PlateProtocol:
    F_N: float                    # normal load [N] (2550 N)
    t_ramp: float = 0.5           # load ramp [s] (SPEC S:495 design decision)
    t_I_end: float = 2.5          # end of phase I [s]
    u_shear: float = 0.1          # pull speed [m/s] (100 mm/s)
    t_shear_ramp: float = 0.1     # speed ramp [s]
    t_II_end: float = 2.75        # end of the peak-traction window [s]
    t_end: float = 5.4            # end of the run [s]
    window: float = 0.1           # averaging window of the sinkage metrics [s]
    smooth: float = 0.025         # moving average before the peak-traction maximum [s]
    max_contact_loss: float = 0.2  # no plate contact for longer in phase II/III: fault
    f_pull_max: float = float("inf")  # Eq. 4 limit |lambda| <= f_pull_max on the pull motor


class ExperimentFault(RuntimeError):
    """The run cannot yield metrics (the plate lost contact, or F_N = 0)."""


def run_plate_test(bed: "D.Bed", plate: int, proto: PlateProtocol, dt: float, z_datum: float, record_every: int = 1):
    """Drive plate `plate` of `bed` through phases I-III; returns the per-step series (dict of
    arrays).  z_datum: plate reference height at which the grouser tips touch the surface.  The
    applied load is the force-axis target; the plate's own weight is not added (gravity acts on
    particles only), so F_N is the whole vertical load."""
    if not proto.F_N > 0:
        raise ExperimentFault("F_N <= 0: the traction coefficient is undefined (SPEC S:476)")
    lost = 0.0
    n_steps = int(np.ceil(proto.t_end / dt - 1e-9))     # the series covers [0, t_end]
    n_I = int(np.ceil(proto.t_I_end / dt - 1e-9))
    cols = {k: [] for k in ("t", "sinkage", "F_N_applied", "F_N_measured", "F_T", "traction", "plate_x", "n_contacts")}
    bed.drive_plate(plate, 0, D.AXIS_LOCKED, 0.0)
    for s in range(n_steps):
        t0 = s * dt
        if s < n_I:
            F = proto.F_N * min(1.0, (t0 + dt) / proto.t_ramp) if proto.t_ramp > 0 else proto.F_N
            bed.drive_plate(plate, 2, D.AXIS_FORCE, -F)          # downward load on a force axis
        elif s == n_I:
            bed.drive_plate(plate, 2, D.AXIS_FORCE, -proto.F_N)
            bed.drive_plate(plate, 0, D.AXIS_VELOCITY, proto.u_shear, proto.t_shear_ramp,
                            -proto.f_pull_max, proto.f_pull_max)
        rep = bed.step(1)
        if s % record_every:
            continue
        g = bed.get_plate(plate)
        F_app = proto.F_N * min(1.0, (t0 + dt) / proto.t_ramp) if (s < n_I and proto.t_ramp > 0) else proto.F_N
        cols["t"].append(rep["time"])
        cols["sinkage"].append(z_datum - g["pos"][2])
        cols["F_N_applied"].append(F_app)
        cols["F_N_measured"].append(g["force"][2])
        F_T = g["motor_force"][0]                                   # the pull motor's force
        cols["F_T"].append(F_T)
        cols["traction"].append(F_T / F_app if F_app > 0 else np.nan)
        cols["plate_x"].append(g["pos"][0])
        cols["n_contacts"].append(g["n_contacts"])
        if s >= n_I:                                               # SPEC S:474 experiment fault
            lost = lost + dt * record_every if g["n_contacts"] == 0 else 0.0
            if lost > proto.max_contact_loss:
                raise ExperimentFault(f"plate lost contact for > {proto.max_contact_loss} s at t = {rep['time']:.4f} s")
    return {k: np.asarray(v, dtype=float) for k, v in cols.items()}


def surface_datum(pos, radius, center_xy, half_xy, cell=None):
    """Sinkage datum (SPEC S:498 design decision): mean height of the top particle surface under
    the plate footprint -- the footprint binned into square columns of side 2 r_max, the column
    top = max(z + r) of the particles whose centres lie in it, the datum = mean column top."""
    pos, radius = np.asarray(pos, float), np.asarray(radius, float)
    cell = 2.0 * radius.max() if cell is None else cell
    lo = np.asarray(center_xy, float) - np.asarray(half_xy, float)
    hi = np.asarray(center_xy, float) + np.asarray(half_xy, float)
    m = np.all((pos[:, :2] >= lo) & (pos[:, :2] < hi), axis=1)
    if not m.any():
        raise ValueError("no particle under the plate footprint")
    ij = np.floor((pos[m, :2] - lo) / cell).astype(np.int64)
    top = pos[m, 2] + radius[m]
    cols = {}
    for (i, j), z in zip(map(tuple, ij), top):
        cols[(i, j)] = max(cols.get((i, j), -np.inf), z)
    return float(np.mean(list(cols.values())))


def write_csv(path, series):
    """Per-run CSV (SPEC S:507 external interface; columns of the recorded series)."""
    keys = list(series)
    with open(path, "w") as f:
        f.write(",".join(keys) + "\n")
        for row in zip(*(series[k] for k in keys)):
            f.write(",".join(repr(float(v)) for v in row) + "\n")


def _moving_average(t, y, width):
    """Centred moving average over a time window |t' - t| <= width/2 (a windowed mean, so it does
    not depend on the sampling rate)."""
    c = np.concatenate(([0.0], np.cumsum(y)))
    lo = np.searchsorted(t, t - 0.5 * width, side="left")
    hi = np.searchsorted(t, t + 0.5 * width, side="right")
    return (c[hi] - c[lo]) / (hi - lo)


def extract_metrics(series, proto: PlateProtocol):
    """SPEC S:478-482 (PAPER §4.1-4.2): static sinkage = mean sinkage over the last `window` of
    phase I; peak traction = max of the `smooth`-averaged traction in [t_I_end, t_II_end];
    average traction = mean traction over [t_I_end, t_end]; dynamic sinkage = mean sinkage over
    the last `window` of the run."""
    t = np.asarray(series["t"], float)
    if len(t) == 0 or t[-1] < proto.t_end - 1e-12 * max(1.0, proto.t_end) or t[0] > proto.t_I_end - proto.window:
        raise ValueError("series shorter than the metric windows")
    s, tr = np.asarray(series["sinkage"], float), np.asarray(series["traction"], float)
    w1 = (t > proto.t_I_end - proto.window) & (t <= proto.t_I_end)
    w2 = t > t[-1] - proto.window
    sh = t > proto.t_I_end
    pk = sh & (t <= proto.t_II_end)
    trs = _moving_average(t[sh], tr[sh], proto.smooth)
    return {
        "static_sinkage": float(s[w1].mean()),
        "dynamic_sinkage": float(s[w2].mean()),
        "peak_traction": float(trs[pk[sh]].max()),
        "avg_traction": float(tr[sh].mean()),
        # SPEC S:519 open question: dynamic sinkage read as end-of-run sinkage; the growth after
        # phase I is emitted beside it
        "dynamic_sinkage_growth": float(s[w2].mean() - s[w1].mean()),
    }


def normalized_errors(m, m_ref, h_grouser, F_N_max, F_N=None):
    """PAPER §4.3: sinkage errors normalised by the grouser depth,
    traction errors as force differences F_T - F_T,ref = (coefficient difference) F_N normalised
    by the maximum normal load; aggregate = mean of the four absolute values."""
    F_N = F_N_max if F_N is None else F_N
    e = {
        "static_sinkage": (m["static_sinkage"] - m_ref["static_sinkage"]) / h_grouser,
        "dynamic_sinkage": (m["dynamic_sinkage"] - m_ref["dynamic_sinkage"]) / h_grouser,
        "peak_traction": (m["peak_traction"] - m_ref["peak_traction"]) * F_N / F_N_max,
        "avg_traction": (m["avg_traction"] - m_ref["avg_traction"]) * F_N / F_N_max,
    }
    e["aggregate"] = float(np.mean([abs(v) for v in e.values()]))
    return e
