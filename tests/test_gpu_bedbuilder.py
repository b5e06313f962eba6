"""Bed builder on the GPU (PAPER §3.1): small uniform and
layer-refined beds emitted, trimmed, relaxed at reduced friction and settled at full friction
with the paper's material (rho 2200, E 1 GPa, nu 0.15, mu 0.3 / 0.02); SPEC invariants: every
centre inside the container, every diameter within [0.9, 1.1] d_n of its layer, post-settle
overlap <= 0.02 d, settled (KE and speed), layers where the schedule puts them, determinism."""
import numpy as np
import pytest

from paper_2501_05300_b200 import bedbuilder as BB
from paper_2501_05300_b200.protocol import surface_datum

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def check_bed(out, spec):
    x, r = out["pos"], out["radius"]
    L = np.asarray(spec.dims)
    assert len(r) > 50
    assert np.all(x > 0) and np.all(x < L)
    sched = list(reversed(out["schedule"]))                            # layer 0 = bottom band
    dn = np.array([b[0] for b in sched])[out["layer"]]
    assert np.all(2 * r >= (1 - spec.jitter) * dn * (1 - 1e-12))
    assert np.all(2 * r <= (1 + spec.jitter) * dn * (1 + 1e-12))
    au = BB.audit_bed(x, r, spec.dims, 2.2 * (spec.d_max or spec.d_min), spec.material["density"],
                      layer=out["layer"], schedule=out["schedule"])
    assert au["max_overlap_ratio"] <= 0.02
    assert au["mixing"] <= 0.05
    assert np.abs(out["vel"]).max() < 2e-3                              # settled
    return au


def test_uniform_bed_and_determinism():
    spec = BB.BedSpec(dims=(0.08, 0.08, 0.06), d_min=0.01, seed=3)
    a = BB.build_bed(spec)
    au = check_bed(a, spec)
    # bulk density below the surface: ~1400 kg/m^3 for the paper's beds (phi ~ 0.64);
    # this 8-diameter box with walls packs looser
    H = surface_datum(a["pos"], a["radius"], (0.04, 0.04), (0.04, 0.04), cell=0.02)
    rho_b = (2200.0 * 4 / 3 * np.pi * a["radius"] ** 3).sum() / (0.08 * 0.08 * H)
    print("uniform: n", len(a["radius"]), "t_sim", a["t_sim"], "dt", a["dt"], "surface", H, "bulk density", rho_b)
    assert H > 0.045
    assert 1000.0 < rho_b < 1500.0
    b = BB.build_bed(spec)
    assert np.array_equal(a["pos"], b["pos"]) and np.array_equal(a["radius"], b["radius"])


def test_layered_bed():
    # r = 1.2, eta = 2: gamma = (r - 1)/(r eta) = 0.083, four layers 6 -> 10.4 mm; the
    # paper excludes aggressive gamma ~ 1 for size mixing, at gamma 0.33 this bed mixes 16 %
    spec = BB.BedSpec(dims=(0.1, 0.1, 0.06), d_min=0.006, d_max=0.0104, r=1.2, eta=2.0, seed=4)
    out = BB.build_bed(spec)
    au = check_bed(out, spec)
    print("layered: n", len(out["radius"]), "t_sim", out["t_sim"], "mixing", au["mixing"],
          "per layer", np.bincount(out["layer"]))
    # the finest particles are on top, the coarsest at the bottom
    z_by_layer = [out["pos"][out["layer"] == k, 2].mean() for k in range(out["layer"].max() + 1)]
    assert all(z_by_layer[k] < z_by_layer[k + 1] for k in range(len(z_by_layer) - 1))


def test_builder_matches_the_oracle_pipeline():
    """SURVEY NEXT-2 parity: one tiny two-layer spec built by the same host pipeline
    through libdem (GPU) and through the fp64 oracle (tests/oracle_bed.OracleBed).  Emission and
    trimming follow the settled states, which part ways chaotically (rounding), so the beds are
    compared by the quantities the paper's procedure controls: particles per layer (within 5 %),
    the bulk density below the surface (within 3 %), the mixing metric (within 0.02) and the
    overlap bound of both (<= 2 % of d)."""
    from tests.oracle_bed import OracleBed
    spec = BB.BedSpec(dims=(0.05, 0.05, 0.045), d_min=0.008, d_max=0.012, r=1.5, eta=1.5, seed=5)
    g = BB.build_bed(spec)
    o = BB.build_bed(spec, bed_factory=lambda **kw: OracleBed(**kw))

    def summary(out):
        x, r = out["pos"], out["radius"]
        au = BB.audit_bed(x, r, spec.dims, 2.2 * spec.d_max, spec.material["density"], layer=out["layer"],
                          schedule=out["schedule"])
        H = surface_datum(x, r, (0.025, 0.025), (0.025, 0.025), cell=0.02)
        rho_b = (spec.material["density"] * 4 / 3 * np.pi * r[x[:, 2] < H] ** 3).sum() / (0.05 * 0.05 * H)
        return dict(n_layer=np.bincount(out["layer"]), rho_b=rho_b, mixing=au["mixing"], overlap=au["max_overlap_ratio"])

    sg, so = summary(g), summary(o)
    print("gpu", sg, "oracle", so)
    assert len(sg["n_layer"]) == len(so["n_layer"]) >= 2
    np.testing.assert_allclose(sg["n_layer"], so["n_layer"], rtol=0.05)
    assert sg["rho_b"] == pytest.approx(so["rho_b"], rel=0.03)
    assert abs(sg["mixing"] - so["mixing"]) <= 0.02
    assert sg["overlap"] <= 0.02 and so["overlap"] <= 0.02
