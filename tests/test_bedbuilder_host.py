"""Bed builder host logic (PAPER §2.1, §3.1):
the layer schedule against the paper's geometric sum, the density audit against exact mass
accounting, the emitter plane's geometry."""
import numpy as np
import pytest

from paper_2501_05300_b200 import bedbuilder as BB


def test_layer_schedule_geometric_sum():
    # d_n = r d_{n-1}, thickness eta d_n, bottom of layer n at depth
    # z_n = eta d_0 (r^{n+1} - 1)/(r - 1), and d_n = d_0/r + (r - 1)/(r eta) z_n (gamma = (r-1)/(r eta))
    d0, r, eta = 8.5e-3, 1.2, 1.0
    sched = BB.layer_schedule(d0, 30e-3, r, eta, 0.6)
    for n, (d, top, bot) in enumerate(sched[:-1]):
        assert d == pytest.approx(d0 * r ** n, rel=1e-12)
        assert bot == pytest.approx(eta * d0 * (r ** (n + 1) - 1) / (r - 1), rel=1e-12)
        assert d == pytest.approx(d0 / r + (r - 1) / (r * eta) * bot, rel=1e-12)
        assert bot - top == pytest.approx(eta * d, rel=1e-12)
    # the coarsest layer is capped at d_max and runs to the bottom of the container
    assert sched[-1][0] <= 30e-3 and sched[-1][2] == pytest.approx(0.6)
    assert all(sched[k][2] == sched[k + 1][1] for k in range(len(sched) - 1))


def test_layer_schedule_uniform_and_degenerate():
    assert BB.layer_schedule(15e-3, 15e-3, 1.0, 1.0, 0.3) == [(15e-3, 0.0, 0.3)]
    assert BB.layer_schedule(15e-3, 30e-3, 1.0, 1.0, 0.3) == [(15e-3, 0.0, 0.3)]
    assert BB.layer_schedule(15e-3, 15e-3, 1.0, 1.0, 0.0) == []          # empty world
    with pytest.raises(ValueError):
        BB.layer_schedule(15e-3, 10e-3, 1.2, 1.0, 0.3)


def test_audit_mass_accounting():
    rho = 2200.0
    dims = (0.1, 0.1, 0.1)
    # one sphere well inside a cell: that cell holds its whole mass
    out = BB.audit_bed([[0.025, 0.025, 0.025]], [0.01], dims, 0.05, rho)
    m = rho * 4 / 3 * np.pi * 0.01 ** 3
    assert out["density"][0, 0, 0] * 0.05 ** 3 == pytest.approx(m, rel=1e-12)
    assert out["density"].sum() * 0.05 ** 3 == pytest.approx(m, rel=1e-12)
    # a sphere centred on a cell face splits exactly in half (symmetric quadrature)
    out = BB.audit_bed([[0.05, 0.025, 0.025]], [0.01], dims, 0.05, rho)
    assert out["density"][0, 0, 0] == pytest.approx(out["density"][1, 0, 0], rel=1e-12)
    # vacuum -> 0; total mass conserved for a random set
    rng = np.random.default_rng(1)
    pos = rng.uniform(0.01, 0.09, (200, 3))
    rad = rng.uniform(0.003, 0.006, 200)
    out = BB.audit_bed(pos, rad, dims, 0.025, rho)
    assert out["density"].sum() * 0.025 ** 3 == pytest.approx((rho * 4 / 3 * np.pi * rad ** 3).sum(), rel=1e-12)
    assert BB.audit_bed(np.zeros((0, 3)), np.zeros(0), dims, 0.025, rho)["mean"] == 0.0
    with pytest.raises(ValueError):
        BB.audit_bed(pos, rad, dims, 0.005, rho)                        # cell < d_max


def test_audit_overlap_and_mixing():
    pos = np.array([[0.02, 0.02, 0.01], [0.02 + 0.0196, 0.02, 0.01]])
    out = BB.audit_bed(pos, [0.01, 0.01], (0.1, 0.1, 0.1), 0.025, 2200.0, layer=np.array([0, 0]),
                       schedule=[(0.01, 0.0, 0.05), (0.02, 0.05, 0.1)])
    assert out["max_overlap_ratio"] == pytest.approx(0.0004 / 0.02, rel=1e-9)
    assert out["mixing"] == 0.0                                       # both in the bottom band
    out = BB.audit_bed(pos, [0.01, 0.01], (0.1, 0.1, 0.1), 0.025, 2200.0, layer=np.array([1, 0]),
                       schedule=[(0.01, 0.0, 0.05), (0.02, 0.05, 0.1)])
    assert out["mixing"] == 0.5                                       # one is far below its top band


def test_emitter_plane_no_overlap_inside_container():
    spec = BB.BedSpec(dims=(0.1, 0.08, 0.1), d_min=0.01)
    rng = np.random.default_rng(3)
    p, rad, v, g = BB._emit_plane(spec, rng, 0.01, 0.05, (0.0, 0.0), (0.1, 0.08), 7)
    assert len(p) > 10 and g[0] == 7 and np.all(np.diff(g) == 1)
    assert np.all(rad >= 0.45 * 0.01 - 1e-15) and np.all(rad <= 0.55 * 0.01 + 1e-15)
    assert np.all(p[:, 0] - rad > 0) and np.all(p[:, 0] + rad < 0.1)
    assert np.all(p[:, 1] - rad > 0) and np.all(p[:, 1] + rad < 0.08)
    d = np.linalg.norm(p[:, None, :] - p[None, :, :], axis=2) + np.eye(len(p))
    assert np.all(d > rad[:, None] + rad[None, :])
    assert np.all(v[:, 2] < 0)


def test_build_logic_on_the_oracle():
    """The whole build pipeline (emission planes, settling, trimming, friction restored) driven
    through the fp64 oracle on a tiny container: SPEC invariants hold and the bed fills it."""
    from tests.oracle_bed import OracleBed
    spec = BB.BedSpec(dims=(0.05, 0.05, 0.035), d_min=0.01, seed=2)
    out = BB.build_bed(spec, bed_factory=lambda **kw: OracleBed(**kw))
    x, r = out["pos"], out["radius"]
    assert len(r) >= 20
    assert np.all(x > 0) and np.all(x < np.asarray(spec.dims))
    assert np.all(2 * r >= 0.9 * 0.01 - 1e-15) and np.all(2 * r <= 1.1 * 0.01 + 1e-15)
    assert np.abs(out["vel"]).max() < 1e-3
    from paper_2501_05300_b200.protocol import surface_datum
    assert surface_datum(x, r, (0.025, 0.025), (0.025, 0.025), cell=0.02) > 0.035 - 1.05 * 0.01 - 0.01
