"""Pins of the fp64 oracle against what the paper, SPEC worked examples and mathematics fix.

Each test names the passage it pins.  None of these retypes the oracle's code path: they use
closed forms (Hertz/linear-dashpot collisions, incline dynamics, free flight), printed worked
examples (tests/golden/spec_examples.json), library routines (scipy distance matrices, dense
linear solves of the LCP by active-set enumeration) or conservation laws.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.distance import cdist
from scipy.special import beta as Beta

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def sig(x, digits):
    return float(f"{x:.{digits - 1}e}")


# ---------------------------------------------------------------- material / planner pins

def test_mass_inertia_spec(oracle_mod):
    for ex in GOLD["mass_inertia"]:
        m, I = oracle_mod.mass_inertia(ex["d"], ex["rho"])
        assert sig(m, ex["digits"]) == pytest.approx(ex["m"], rel=1e-12), ex["cite"]
        if "I" in ex:
            assert I == pytest.approx(ex["I"], rel=1e-12)
    # scaling invariant: m(2d) = 8 m(d), I(2d) = 32 I(d)
    rng = np.random.default_rng(1)
    for d in rng.uniform(1e-3, 5e-2, 10):
        m1, I1 = oracle_mod.mass_inertia(d, 2600.0)
        m2, I2 = oracle_mod.mass_inertia(2 * d, 2600.0)
        assert m2 == pytest.approx(8 * m1, rel=1e-12) and I2 == pytest.approx(32 * I1, rel=1e-12)


def test_contact_params_spec(oracle_mod):
    ex = GOLD["contact_params"][0]
    Es, ds, kn, eps = oracle_mod.contact_params(ex["d"], ex["d"], ex["E"], ex["E"], ex["nu"], ex["nu"])
    assert sig(Es, 4) == ex["Estar"] and sig(kn, 4) == ex["kn"] and sig(eps, 4) == ex["eps_n"]
    assert ds == pytest.approx(ex["dstar"], rel=1e-12)
    # identical materials: E* = E/(2(1-nu^2)); flat tool d* = d; symmetry
    assert Es == pytest.approx(1e9 / (2 * (1 - 0.15**2)), rel=1e-14)
    assert oracle_mod.contact_params(8.5e-3, 0.0, 1e9, 1e9, .15, .15)[1] == pytest.approx(8.5e-3, rel=1e-14)
    a = oracle_mod.contact_params(3e-3, 7e-3, 1e9, 2e8, .15, .3)
    b = oracle_mod.contact_params(7e-3, 3e-3, 2e8, 1e9, .3, .15)
    assert a == pytest.approx(b, rel=1e-14)


def test_planner_spec(oracle_mod):
    for ex in GOLD["profile"]:
        d = oracle_mod.profile_diameter(ex["d_min"], ex["d_max"], ex["gamma"], ex["z"])
        assert d == pytest.approx(ex["d"], rel=1e-12), ex["cite"]
    ls = GOLD["layer_schedule"]
    d, z = oracle_mod.layer_schedule(ls["d_min"], ls["d_max"], ls["r"], ls["eta"])
    assert np.round(d * 1e3, 2).tolist() == ls["d_mm"]
    assert z[0] * 1e3 == pytest.approx(ls["z0_mm"]) and z[1] * 1e3 == pytest.approx(ls["z1_mm"])
    # unclamped layers lie on d_n = d_0/r + gamma z_n with gamma = (r-1)/(r eta)
    g = (ls["r"] - 1) / (ls["r"] * ls["eta"])
    assert round(g, 4) == ls["gamma"]
    np.testing.assert_allclose(d[:-1], ls["d_min"] / ls["r"] + g * z[:-1], rtol=1e-12)
    ge = GOLD["gamma_r_eta"]
    assert round((ge["r"] - 1) / (ge["r"] * ge["eta"]), 4) == ge["gamma"]
    for ex in GOLD["network_length"]:
        nd = oracle_mod.contact_network_length(ex["d_min"], ex["d_max"], ex["r"], ex["eta"], ex["h"])
        assert round(nd, 1) == ex["n_d"], ex["cite"]
    for ex in GOLD["iterations"]:
        assert oracle_mod.solver_iterations(ex["n_d"], ex["eps"]) == ex["N_it"], ex["cite"]
    for ex in GOLD["timestep"]:
        dt = oracle_mod.planned_timestep(ex["d"], ex["eps"], ex["rho"], ex["sigma"])
        assert sig(dt, 3) == pytest.approx(ex["dt"]), ex["cite"]
        assert abs(dt - ex["paper_dt"]) / ex["paper_dt"] < 0.04   # Table 3 within 4 %
        # closed form dt = d sqrt(eps rho / 6 sigma)
        assert dt == pytest.approx(ex["d"] * math.sqrt(ex["eps"] * ex["rho"] / (6 * ex["sigma"])), rel=1e-12)


# ---------------------------------------------------------------- detection pins

def _world(oracle_mod, x, r, gid=None, v=None, walls=(), plates=()):
    n = len(r)
    return oracle_mod.OracleWorld(x, np.zeros((n, 3)) if v is None else v, np.zeros((n, 3)), r,
                                  np.arange(n) if gid is None else gid, walls=walls, plates=plates)


def test_detect_examples(oracle_mod):
    # empty world
    c, nd = _world(oracle_mod, np.zeros((0, 3)), np.zeros(0)).detect()
    assert len(c) == 0 and nd == 0
    # spheres d=10 mm, centres 9 mm apart -> delta = 1 mm along the centre line
    c, _ = _world(oracle_mod, [[0, 0, 0], [0, 9e-3, 0]], [5e-3, 5e-3]).detect()
    assert len(c) == 1 and c["delta"][0] == pytest.approx(1e-3, rel=1e-12)
    np.testing.assert_allclose(c["n"][0], [0, 1, 0], atol=1e-15)
    # distance 0.9 (r_a + r_b) is a contact; 1.0001 is not
    c, _ = _world(oracle_mod, [[0, 0, 0], [0.9 * 5e-3, 0, 0]], [2e-3, 3e-3]).detect()
    assert len(c) == 1
    c, _ = _world(oracle_mod, [[0, 0, 0], [1.0001 * 5e-3, 0, 0]], [2e-3, 3e-3]).detect()
    assert len(c) == 0
    # sphere d = 10 mm with its centre 4 mm above a plane -> delta = 1 mm
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    c, _ = _world(oracle_mod, [[0.1, 0.2, 4e-3]], [5e-3], walls=floor).detect()
    assert len(c) == 1 and c["delta"][0] == pytest.approx(1e-3, rel=1e-12)
    np.testing.assert_allclose(c["n"][0], [0, 0, -1])
    assert int(c["key"][0]) & 0xFFFFFFFF == oracle_mod.WALL_KEY_BASE + 4   # floor = wall 4 (-z)
    # coincident centres are flagged and skipped
    c, nd = _world(oracle_mod, [[0, 0, 0], [0, 0, 0], [1, 1, 1]], [1e-3, 2e-3, 1e-3]).detect()
    assert len(c) == 0 and nd == 1
    # orientation: n from smaller gid to larger gid, antisymmetric under relabelling
    x = [[0, 0, 0], [3e-3, 1e-3, 0]]
    c1, _ = _world(oracle_mod, x, [2e-3, 2e-3], gid=[5, 9]).detect()
    c2, _ = _world(oracle_mod, x, [2e-3, 2e-3], gid=[9, 5]).detect()
    np.testing.assert_allclose(c1["n"][0], -c2["n"][0], rtol=0, atol=0)
    assert c1["key"][0] == c2["key"][0] == (5 << 32 | 9)


@pytest.mark.parametrize("seed,n", [(3, 400), (4, 1000)])
def test_pair_set_vs_distance_matrix(oracle_mod, seed, n):
    """Pair set equals the all-pairs distance-matrix oracle, polydisperse 8x."""
    import synth
    b = synth.random_cloud(n, (0, 0, 0), (0.08, 0.08, 0.08), 1e-3, 8e-3, seed, loguniform=True)
    c, _ = _world(oracle_mod, b.x, b.r, gid=b.gid).detect()
    D = cdist(b.x, b.x)
    S = b.r[:, None] + b.r[None, :]
    ii, jj = np.nonzero(np.triu(D < S, 1))
    ga, gb = np.minimum(b.gid[ii], b.gid[jj]), np.maximum(b.gid[ii], b.gid[jj])
    want = np.sort((ga.astype(np.uint64) << np.uint64(32)) | gb.astype(np.uint64))
    np.testing.assert_array_equal(c["key"], want)
    # overlap depth per pair = r_a + r_b - |x_b - x_a|
    inv = np.argsort(b.gid)
    a_i = inv[(c["key"] >> np.uint64(32)).astype(np.int64)]
    b_i = inv[(c["key"] & np.uint64(0xFFFFFFFF)).astype(np.int64)]
    np.testing.assert_allclose(c["delta"], S[a_i, b_i] - D[a_i, b_i], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(np.linalg.norm(c["n"], axis=1), 1.0, rtol=1e-14)


def test_contacts_of_vs_distance_matrix(oracle_mod):
    """or_contacts_of (the reference of the full-size sampled GPU checks): the contacts of a sample
    of particles equal the distance-matrix pairs that involve a sampled particle, plus the walls
    whose signed distance is below the radius; keys deduplicated (pairs of two sampled particles
    once) and sorted, depths r_a + r_b - d."""
    import synth
    b = synth.random_cloud(800, (0, 0, 0), (0.06, 0.06, 0.06), 1e-3, 6e-3, 17, loguniform=True)
    lo, hi = (0.0, 0.0, 0.0), (0.06, 0.06, 0.06)
    W = oracle_mod.OracleWorld(b.x, b.v, b.w, b.r, b.gid, walls=oracle_mod.box_walls(lo, hi))
    sample = np.random.default_rng(5).choice(b.n, 60, replace=False)
    got = W.contacts_of(sample)
    D = cdist(b.x, b.x)
    S = b.r[:, None] + b.r[None, :]
    ii, jj = np.nonzero(np.triu(D < S, 1))
    insample = np.zeros(b.n, bool)
    insample[sample] = True
    keep = insample[ii] | insample[jj]
    ga, gb = np.minimum(b.gid[ii[keep]], b.gid[jj[keep]]), np.maximum(b.gid[ii[keep]], b.gid[jj[keep]])
    want = list((ga.astype(np.uint64) << np.uint64(32)) | gb.astype(np.uint64))
    for i in sample:                       # walls: key (gid, 2^32 - 16 + w), w = -x,+x,-y,+y,-z,+z
        for ax in range(3):
            for side in range(2):
                s_ = b.x[i, ax] - lo[ax] if side == 0 else hi[ax] - b.x[i, ax]
                if s_ < b.r[i]:
                    want.append((np.uint64(b.gid[i]) << np.uint64(32)) | np.uint64(0xFFFFFFF0 + 2 * ax + side))
    want = np.sort(np.array(want, dtype=np.uint64))
    np.testing.assert_array_equal(got["key"], want)
    assert len(got) > 60
    pp = (got["key"] & np.uint64(0xFFFFFFFF)) < np.uint64(0xFFFFF000)
    inv = np.argsort(b.gid)
    a_i = inv[(got["key"][pp] >> np.uint64(32)).astype(np.int64)]
    b_i = inv[(got["key"][pp] & np.uint64(0xFFFFFFFF)).astype(np.int64)]
    np.testing.assert_allclose(got["delta"][pp], S[a_i, b_i] - D[a_i, b_i], rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("case", ["cloud8x", "jammed_bands", "coincident", "sparse"])
def test_binning_mode_equals_brute_force(oracle_mod, case):
    """SURVEY §8(c) binning mode: the cell-list pair enumeration returns the brute force's
    contacts bit for bit (keys, normals, depths, degenerate count), and a whole step with it
    (detection inside or_step) is bit-identical.  Pinned to the distance matrix through the
    brute force (test_pair_set_vs_distance_matrix)."""
    import synth
    if case == "cloud8x":
        b = synth.random_cloud(1500, (0, 0, 0), (0.1, 0.1, 0.1), 1e-3, 8e-3, 11, loguniform=True, v_scale=0.1)
    elif case == "jammed_bands":
        b = synth.banded_bed((0.03, 0.03, 0.03), [(0.0, 0.01, 1e-3), (0.01, 0.03, 2.5e-3)], 12, spacing=2.0)
    elif case == "coincident":    # duplicated centres: degenerate pairs counted the same way
        b = synth.random_cloud(300, (0, 0, 0), (0.03, 0.03, 0.03), 1e-3, 2e-3, 13)
        b.x[1::7] = b.x[0:-1:7][: len(b.x[1::7])]
    else:                         # sparse pairs in a 1 m cube: the cell-size cap (cells doubled)
        rng = np.random.default_rng(14)
        c = rng.uniform(0, 1, (150, 3))
        x = np.concatenate([c, c + rng.uniform(-1.5e-3, 1.5e-3, (150, 3))])
        b = synth.Bed(x=x, r=np.full(300, 1e-3), v=np.zeros((300, 3)), w=np.zeros((300, 3)),
                      gid=rng.permutation(300).astype(np.uint32), box_lo=(0, 0, 0), box_hi=(1, 1, 1))
    try:
        oracle_mod.set_binning(False)
        c0, d0 = _world(oracle_mod, b.x, b.r, gid=b.gid).detect()
        oracle_mod.set_binning(True)
        c1, d1 = _world(oracle_mod, b.x, b.r, gid=b.gid).detect()
        assert d0 == d1 and len(c0) == len(c1) > 0
        for k in ("key", "n", "delta"):
            assert np.array_equal(c0[k], c1[k]), k
        if case == "cloud8x":
            p = oracle_mod.make_params(h=1e-4, n_it=20)
            out = []
            for on in (False, True):
                oracle_mod.set_binning(on)
                W = oracle_mod.OracleWorld(b.x, b.v, b.w, b.r, b.gid)
                W.step(p, 2)
                out.append((W.x.copy(), W.v.copy(), W.w.copy()))
            for u, v in zip(out[0], out[1]):
                assert np.array_equal(u, v)
    finally:
        oracle_mod.set_binning(False)


def test_plate_box_closest_point_dense_sampling(oracle_mod):
    """Sphere vs grouser box edge/corner: delta and normal match a dense sampling of the box
    surface."""
    lo, hi = np.array([0.0, 0.0, 0.0]), np.array([0.0255, 0.05, 0.043])
    P = oracle_mod.make_plate([lo], [hi], pos=(0, 0, 0), mass=1.0)
    h = 2e-5
    ax = [np.arange(lo[k], hi[k] + h / 2, h) for k in range(3)]
    faces = []
    for k in range(3):
        o = [a for j, a in enumerate(ax) if j != k]
        A, B = np.meshgrid(*o, indexing="ij")
        for val in (lo[k], hi[k]):
            pts = np.empty((A.size, 3))
            pts[:, [j for j in range(3) if j != k]] = np.stack([A.ravel(), B.ravel()], 1)
            pts[:, k] = val
            faces.append(pts)
    surf = np.concatenate(faces)
    rng = np.random.default_rng(7)
    for X in [np.array([-1e-3, -1e-3, 0.044]), np.array([0.027, 0.02, -1.5e-3]), np.array([0.0265, 0.051, 0.044])]:
        r = 3e-3
        c, _ = _world(oracle_mod, [X], [r], plates=[P]).detect()
        d = np.linalg.norm(surf - X, axis=1)
        k = np.argmin(d)
        assert len(c) == 1
        assert c["delta"][0] == pytest.approx(r - d[k], abs=2 * h)
        np.testing.assert_allclose(c["n"][0], (surf[k] - X) / d[k], atol=0.02)
    del rng


# ---------------------------------------------------------------- dynamics pins

R0, RHO = 3e-3, 2600.0


def _headon(oracle_mod, v0, h, r=R0, max_steps=400000, **kw):
    x = np.array([[0, 0, 0], [2 * r + 1e-12, 0, 0]])
    v = np.array([[v0 / 2, 0, 0], [-v0 / 2, 0, 0]])
    W = _world(oracle_mod, x, [r, r], v=v)
    p = oracle_mod.make_params(h=h, n_it=kw.pop("n_it", 30), v_imp=kw.pop("v_imp", 1e30), g=(0, 0, 0),
                               mu_t=0, mu_r=0, **kw)
    n_force, touched, dmax = 0, False, 0.0
    for _ in range(max_steps):
        c, _, _ = W.step(p)
        if len(c):
            touched = True
            dmax = max(dmax, c["delta"][0])
            if c["P"][0, 0] > 0:
                n_force += 1
        elif touched:
            break
    e = (W.v[1, 0] - W.v[0, 0]) / v0
    return n_force * h, e, dmax, W


def test_headon_hertz_closed_form(oracle_mod):
    """Undamped Hertz (tau = 0), no impact stage: delta_max = (5 m* v0^2/(4 k_n))^(2/5),
    t_c = 2 (2/5) B(2/5,1/2) delta_max / v0, e = 1 (P:127-128 mapping, SPOOK P:132)."""
    v0, h = 0.1, 2e-6
    tc, e, dmax, _ = _headon(oracle_mod, v0, h, damp_steps=0.0)
    m, _ = oracle_mod.mass_inertia(2 * R0, RHO)
    Es = 1e7 / (2 * (1 - 0.3**2))
    kn = Es * math.sqrt(R0) / 3.0          # d* = (1/d + 1/d)^-1 = r
    dm = (5 * (m / 2) * v0**2 / (4 * kn)) ** 0.4
    tc_exact = 2 * 0.4 * Beta(0.4, 0.5) * dm / v0
    assert tc == pytest.approx(tc_exact, rel=max(0.005, 2 * h / tc_exact))
    assert dmax == pytest.approx(dm, rel=5e-3)
    assert abs(e - 1.0) < 1e-5


def test_headon_linear_dashpot_closed_form(oracle_mod):
    """Linear model e_H = 1 with SPOOK damping time tau: the no-tension
    Kelvin-Voigt dashpot gives t_c = (pi - atan(2 b w/(w^2 - b^2)))/w and e = exp(-b t_c)."""
    v0, h, klin, damp = 0.1, 2.5e-6, 5e3, 20.0
    tc, e, _, _ = _headon(oracle_mod, v0, h, e_H=1.0, k_lin=klin, damp_steps=damp)
    m, _ = oracle_mod.mass_inertia(2 * R0, RHO)
    ms = m / 2
    tau = damp * h
    b = tau * klin / (2 * ms)
    w = math.sqrt(klin / ms - b * b)
    tc_exact = (math.pi - math.atan(2 * b * w / (w * w - b * b))) / w
    assert tc == pytest.approx(tc_exact, rel=max(0.01, 2 * h / tc_exact))
    assert e == pytest.approx(math.exp(-b * tc_exact), rel=0.01)


def test_free_flight_exact(oracle_mod):
    """No contacts: symplectic Euler x_n = x_0 + n h v_0 + h^2 g n(n+1)/2."""
    h, n = 1e-4, 500
    x0, v0 = np.array([[0.1, 0.2, 0.3]]), np.array([[0.5, -0.2, 1.0]])
    W = _world(oracle_mod, x0, [1e-3], v=v0)
    p = oracle_mod.make_params(h=h)
    W.step(p, n_steps=n)
    g = np.array([0, 0, -9.81])
    np.testing.assert_allclose(W.x, x0 + n * h * v0 + h * h * g * n * (n + 1) / 2, rtol=1e-12)
    np.testing.assert_allclose(W.v, v0 + n * h * g, rtol=1e-12)


def _rest_on_floor(oracle_mod, E=1e9, nu=0.15, rho=2200.0, r=4.25e-3, h=1e-4, steps=300, **kw):
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    W = oracle_mod.OracleWorld([[0, 0, r]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor)
    p = oracle_mod.make_params(h=h, n_it=kw.pop("n_it", 20), E=E, nu=nu, rho=rho, **kw)
    c = None
    for _ in range(steps):
        c, F, T = W.step(p, want_forces=True)
    return W, c, p


def test_statics_resting_particle_hertz(oracle_mod):
    """Resting particle: P_n/h = m g within 1 %; the equilibrium overlap obeys the
    Hertz law k_n delta^(3/2) = m g with k_n = E* sqrt(d*)/3, d* = d for a flat."""
    r = 4.25e-3
    W, c, p = _rest_on_floor(oracle_mod, r=r)
    m, _ = oracle_mod.mass_inertia(2 * r, 2200.0)
    assert c["P"][0, 0] / p.h == pytest.approx(m * 9.81, rel=0.01)
    kn = (1e9 / (2 * (1 - 0.15**2))) * math.sqrt(2 * r) / 3
    assert c["delta"][0] == pytest.approx((m * 9.81 / kn) ** (2 / 3), rel=0.01)
    # g_n = delta^e_H (S:359 worked example): 1 mm -> 1.778e-4
    ex = GOLD["hertz_violation"]
    assert sig(ex["delta"] ** ex["e_H"], 4) == ex["g_n"]


def test_statics_k_stack(oracle_mod):
    """Column of k spheres on a floor: contact forces k mg, (k-1) mg, ...."""
    k, r, h = 4, 4.25e-3, 1e-4
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    x = np.array([[0, 0, r + 2 * r * i] for i in range(k)])
    W = oracle_mod.OracleWorld(x, np.zeros((k, 3)), np.zeros((k, 3)), [r] * k, np.arange(k), walls=floor)
    p = oracle_mod.make_params(h=h, n_it=200, E=1e9, nu=0.15, rho=2200.0)
    for _ in range(400):
        c, _, _ = W.step(p)
    m, _ = oracle_mod.mass_inertia(2 * r, 2200.0)
    keys = c["key"]
    f = {int(kk): c["P"][i, 0] / h for i, kk in enumerate(keys)}
    assert f[(0 << 32) | (oracle_mod.WALL_KEY_BASE + 4)] == pytest.approx(k * m * 9.81, rel=0.01)
    for i in range(k - 1):
        assert f[(i << 32) | (i + 1)] == pytest.approx((k - 1 - i) * m * 9.81, rel=0.01)


@pytest.mark.parametrize("regime", ["static", "rolling", "slipping"])
def test_incline_closed_form(oracle_mod, regime):
    """Sphere on a plane under gravity tilted by theta (R7: rolling radius
    R* = r for walls): static iff tan(theta) <= mu_r; rolling a = 5/7 g (sin - mu_r cos) for
    mu_r < tan <= (7 mu_t - 5 mu_r)/2; slipping a = g (sin - mu_t cos)."""
    mu_t, mu_r, r, h = 0.4, 0.1, 3e-3, 1e-4
    tan = {"static": 0.08, "rolling": 0.5, "slipping": 1.4}[regime]
    th = math.atan(tan)
    g = 9.81
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4, mu_t=mu_t, mu_r=mu_r)
    m, _ = oracle_mod.mass_inertia(2 * r, RHO)
    kn = (1e7 / (2 * (1 - 0.09))) * math.sqrt(2 * r) / 3
    d0 = (m * g * math.cos(th) / kn) ** (2 / 3)
    W = oracle_mod.OracleWorld([[0, 0, r - d0]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor)
    p = oracle_mod.make_params(h=h, n_it=60, mu_t=mu_t, mu_r=mu_r, g=(g * math.sin(th), 0, -g * math.cos(th)))
    vs = []
    for s in range(1500):
        W.step(p)
        vs.append(W.v[0, 0])
    a_meas = (vs[1499] - vs[499]) / (1000 * h)
    if regime == "static":
        assert abs(vs[-1]) < 1e-6
    elif regime == "rolling":
        assert a_meas == pytest.approx(5 / 7 * g * (math.sin(th) - mu_r * math.cos(th)), rel=5e-3)
        assert W.w[0, 1] * r == pytest.approx(W.v[0, 0], rel=5e-3)      # no slip
    else:
        assert a_meas == pytest.approx(g * (math.sin(th) - mu_t * math.cos(th)), rel=5e-3)


def test_newton_impact(oracle_mod):
    """Head-on equal masses, frictionless: after the impact stage u_n+ = -e u_n-, momentum is
    conserved; e = 0 -> common velocity, e = 1 -> exchange."""
    for e in (0.0, 0.5, 1.0):
        x = np.array([[0, 0, 0], [2 * R0 - 1e-10, 0, 0]])
        v = np.array([[0.3, 0, 0], [-0.1, 0, 0]])
        W = _world(oracle_mod, x, [R0, R0], v=v)
        p = oracle_mod.make_params(h=1e-6, n_it=20, e_rest=e, g=(0, 0, 0), mu_t=0, mu_r=0)
        W.step(p)
        assert W.last_report.impact_fired == 1
        un_minus = -0.4
        assert (W.v[1, 0] - W.v[0, 0]) == pytest.approx(-e * un_minus, abs=1e-12)
        assert W.v[:, 0].sum() == pytest.approx(0.2, abs=1e-15)


def _cloud(oracle_mod, seed, n=60, mu=(0.4, 0.1), gravity=(0, 0, 0)):
    import synth
    b = synth.random_cloud(n, (0, 0, 0), (0.03, 0.03, 0.03), 2e-3, 4e-3, seed, v_scale=0.01, w_scale=1.0)
    W = oracle_mod.OracleWorld(b.x, b.v, b.w, b.r, b.gid)
    p = oracle_mod.make_params(h=1e-5, n_it=40, mu_t=mu[0], mu_r=mu[1], g=gravity)
    return W, p, b


def test_momentum_and_angular_momentum_conserved(oracle_mod):
    """Isolated cloud, no gravity: inter-particle impulses cancel and act at a common
    contact point, so sum m v and sum (m x cross v + I w) are conserved exactly in exact arithmetic."""
    W, p, b = _cloud(oracle_mod, 11)
    m = np.array([oracle_mod.mass_inertia(2 * r, p.rho)[0] for r in b.r])
    I = np.array([oracle_mod.mass_inertia(2 * r, p.rho)[1] for r in b.r])
    for _ in range(5):
        P0 = (m[:, None] * W.v).sum(0)
        L0 = (m[:, None] * np.cross(W.x, W.v)).sum(0) + (I[:, None] * W.w).sum(0)
        c, _, _ = W.step(p)
        assert len(c) > 20
        P1 = (m[:, None] * W.v).sum(0)
        L1 = (m[:, None] * np.cross(W.x, W.v)).sum(0) + (I[:, None] * W.w).sum(0)
        scaleP = (m[:, None] * np.abs(W.v)).sum()
        scaleL = (m * np.linalg.norm(W.x, axis=1) * np.linalg.norm(W.v, axis=1)).sum() + (I * np.linalg.norm(W.w, axis=1)).sum()
        np.testing.assert_allclose(P1, P0, atol=1e-13 * scaleP)
        np.testing.assert_allclose(L1, L0, atol=1e-12 * scaleL)


def test_cones_hold(oracle_mod):
    """|P_t| <= mu_t P_n and |P_r| <= mu_r R* P_n after every step."""
    W, p, b = _cloud(oracle_mod, 12, gravity=(0, 0, -9.81))
    inv = {int(g): i for i, g in enumerate(b.gid)}
    for _ in range(3):
        c, _, _ = W.step(p)
        Pn = c["P"][:, 0]
        assert (Pn >= 0).all()
        assert (np.linalg.norm(c["P"][:, 1:4], axis=1) <= p.mu_t * Pn * (1 + 1e-12) + 1e-300).all()
        ia = np.array([inv[int(k >> np.uint64(32))] for k in c["key"]])
        ib = np.array([inv[int(k & np.uint64(0xFFFFFFFF))] for k in c["key"]])
        Rs = b.r[ia] * b.r[ib] / (b.r[ia] + b.r[ib])
        assert (np.linalg.norm(c["P"][:, 4:7], axis=1) <= p.mu_r * Rs * Pn * (1 + 1e-12) + 1e-300).all()
        # tangential impulse lies in the tangent plane
        assert np.abs((c["P"][:, 1:4] * c["n"]).sum(1)).max() <= 1e-12 * max(Pn.max(), 1e-300)


def _lcp_enumeration(A, q):
    """Solve the LCP w = A P + q >= 0, P >= 0, P.w = 0 by active-set enumeration (dense solves)."""
    n = len(q)
    for k in range(n + 1):
        for act in itertools.combinations(range(n), k):
            P = np.zeros(n)
            act = list(act)
            if act:
                P[act] = np.linalg.solve(A[np.ix_(act, act)], -q[act])
            w = A @ P + q
            if (P >= -1e-14).all() and (w >= -1e-12 * (1 + np.abs(q).max())).all():
                return P
    raise AssertionError("no LCP solution")


def test_jacobi_fixed_point_equals_lcp_enumeration(oracle_mod):
    """<= 5 frictionless contacts: the converged Jacobi sweep equals the LCP solution of the
    SPOOK normal rows assembled as a matrix, and warm starting does not change the
    fixed point."""
    r = 3e-3
    h = 1e-5
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    x = np.array([[0, 0, r - 2e-5], [5.9e-3, 0, r - 1e-5], [2.9e-3, 1e-4, r + 5.1e-3]])
    v = np.array([[0.001, 0, -0.002], [0, 0.001, 0], [0, 0, -0.003]])
    n = len(x)
    mk = lambda: oracle_mod.OracleWorld(x, v, np.zeros((n, 3)), [r] * n, np.arange(n), walls=floor)
    p = oracle_mod.make_params(h=h, n_it=20000, mu_t=0, mu_r=0, v_imp=1e30)
    W = mk()
    c, _, _ = W.step(p)
    assert 3 <= len(c) <= 5
    # independent assembly: J (normal rows), M, Sigma-hat, b, v* = v + h g
    m, _ = oracle_mod.mass_inertia(2 * r, p.rho)
    Es = p.E / (2 * (1 - p.nu**2))
    Ups = 1.0 / (1 + 4 * p.damp_steps)
    rows = []
    for i in range(n):
        if x[i, 2] < r:
            rows.append((i, None, np.array([0, 0, -1.0]), r - x[i, 2], r))
        for j in range(i + 1, n):
            d = np.linalg.norm(x[j] - x[i])
            if d < 2 * r:
                rows.append((i, j, (x[j] - x[i]) / d, 2 * r - d, r / 2))
    assert len(rows) == len(c)
    J = np.zeros((len(rows), 3 * n))
    S = np.zeros(len(rows))
    b = np.zeros(len(rows))
    for k, (i, j, nn, dl, Rs) in enumerate(rows):
        J[k, 3 * i:3 * i + 3] = -nn
        if j is not None:
            J[k, 3 * j:3 * j + 3] = nn
        kn = Es * math.sqrt(2 * Rs) / 3
        S[k] = 4 * Ups / (h * h * 1.25 * kn * math.sqrt(dl))
        b[k] = 4 * Ups / h * dl / 1.25 + Ups * (J[k] @ v.ravel())
    vstar = (v + h * np.array([0, 0, -9.81])).ravel()
    A = J @ J.T / m + np.diag(S)
    q = J @ vstar - b
    P = _lcp_enumeration(A, q)
    keys = []
    for (i, j, *_ ) in rows:
        keys.append((i << 32) | (j if j is not None else oracle_mod.WALL_KEY_BASE + 4))
    order = np.argsort(keys)
    np.testing.assert_allclose(c["P"][:, 0], P[order], rtol=1e-6, atol=1e-12 * P.max())
    # warm start from a perturbed history: same fixed point
    W2 = mk()
    hist = c.copy()
    hist["P"][:, 0] *= 1.7
    W2.hist = hist
    c2, _, _ = W2.step(p)
    np.testing.assert_allclose(c2["P"][:, 0], c["P"][:, 0], rtol=1e-6)


def test_gauss_seidel_fixed_point_equals_lcp_enumeration(oracle_mod):
    """Coloured projected Gauss-Seidel (P:134 PGS) converges to the same LCP
    solution of the SPOOK normal rows as the Jacobi iteration: enumeration on the
    configuration of the Jacobi pin, and GS at 200 sweeps already as close as Jacobi at 20,000."""
    r = 3e-3
    h = 1e-5
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    x = np.array([[0, 0, r - 2e-5], [5.9e-3, 0, r - 1e-5], [2.9e-3, 1e-4, r + 5.1e-3]])
    v = np.array([[0.001, 0, -0.002], [0, 0.001, 0], [0, 0, -0.003]])
    n = len(x)
    mk = lambda: oracle_mod.OracleWorld(x, v, np.zeros((n, 3)), [r] * n, np.arange(n), walls=floor)
    cj, _, _ = mk().step(oracle_mod.make_params(h=h, n_it=20000, mu_t=0, mu_r=0, v_imp=1e30))
    cg, _, _ = mk().step(oracle_mod.make_params(h=h, n_it=20000, mu_t=0, mu_r=0, v_imp=1e30, ordering=1))
    np.testing.assert_allclose(cg["P"][:, 0], cj["P"][:, 0], rtol=1e-7)
    c200, _, _ = mk().step(oracle_mod.make_params(h=h, n_it=200, mu_t=0, mu_r=0, v_imp=1e30, ordering=1))
    np.testing.assert_allclose(c200["P"][:, 0], cj["P"][:, 0], rtol=1e-6)


def test_gauss_seidel_single_row_is_exact_after_one_sweep(oracle_mod):
    """one normal row, the LCP solution max(0, -q/(G M^-1 G^T + Sigma)) after ONE
    Gauss-Seidel iteration (sphere resting on a floor, frictionless, no impact stage)."""
    r, h = 3e-3, 1e-5
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    x, v = np.array([[0.0, 0.0, r - 1e-5]]), np.array([[0.0, 0.0, -0.01]])
    W = oracle_mod.OracleWorld(x, v, np.zeros((1, 3)), [r], [0], walls=floor)
    p = oracle_mod.make_params(h=h, n_it=1, mu_t=0, mu_r=0, v_imp=1e30, ordering=1)
    c, _, _ = W.step(p)
    m, _ = oracle_mod.mass_inertia(2 * r, p.rho)
    Es = p.E / (2 * (1 - p.nu**2))
    Ups = 1.0 / (1 + 4 * p.damp_steps)
    dl = 1e-5
    kn = Es * math.sqrt(2 * r) / 3
    S = 4 * Ups / (h * h * 1.25 * kn * math.sqrt(dl))
    # n = -z (particle -> wall): u_n = n.(v_wall - v) = v_z; the bias uses u_n at v^k, the row v* = v^k + h g
    un_star = v[0, 2] + h * -9.81
    b = 4 * Ups / h * dl / 1.25 + Ups * v[0, 2]
    P = max(0.0, -(un_star - b) / (1.0 / m + S))
    assert c["P"][0, 0] == pytest.approx(P, rel=1e-12)


def test_splitmix64_published_values(oracle_mod):
    """The colouring priority is SplitMix64 (Steele, Lea, Flood 2014): with seed 0 its first
    two outputs are 0xE220A8397B1DCDAF and 0x6E789E6AA1B965F4."""
    assert oracle_mod.splitmix64(0) == 0xE220A8397B1DCDAF
    assert oracle_mod.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


@pytest.mark.parametrize("seed", [1, 2])
def test_colouring_is_proper_and_greedy_by_priority(oracle_mod, seed):
    """Checked by properties, not by re-running the algorithm: (1) contacts sharing a particle
    have different colours; (2) every colour below a contact's colour is taken by a conflicting
    contact of higher priority (the defining property of greedy colouring in priority order)."""
    rng = np.random.default_rng(seed)
    n = 60
    a = rng.integers(0, n, 400)
    b = rng.integers(-1, n, 400)
    b = np.where(b == a, -1, b)
    key = np.array([(int(min(x, y)) << 32) | int(max(x, y)) if y >= 0 else (int(x) << 32) | 0xFFFFFFF0
                    for x, y in zip(a, b)], dtype=np.uint64)
    key, idx = np.unique(key, return_index=True)
    a, b = a[idx], b[idx]
    col, ncol = oracle_mod.color_contacts(key, a, b, n)
    assert ncol == col.max() + 1 and ncol > 1
    pri = np.array([oracle_mod.splitmix64(int(k)) for k in key], dtype=object)
    touch = [set() for _ in range(n)]
    for c in range(len(key)):
        touch[a[c]].add(c)
        if b[c] >= 0:
            touch[b[c]].add(c)
    for c in range(len(key)):
        nb = (touch[a[c]] | (touch[b[c]] if b[c] >= 0 else set())) - {c}
        assert all(col[o] != col[c] for o in nb)
        higher = {col[o] for o in nb if (pri[o], -int(key[o])) > (pri[c], -int(key[c]))}
        assert all(q in higher for q in range(col[c]))


def test_gauss_seidel_converges_faster_than_jacobi(oracle_mod):
    """The reason the paper uses PGS: on a 4-stack under gravity, Gauss-Seidel at N
    sweeps is closer to the converged impulses than mass-splitting Jacobi at N sweeps."""
    r, h = 3e-3, 1e-4
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    k = 4
    x = np.array([[0, 0, r + i * (2 * r - 2e-6)] for i in range(k)])
    mk = lambda: oracle_mod.OracleWorld(x, np.zeros((k, 3)), np.zeros((k, 3)), [r] * k, np.arange(k), walls=floor)
    ref, _, _ = mk().step(oracle_mod.make_params(h=h, n_it=20000, v_imp=1e30, ordering=1))
    err = {}
    for o in (0, 1):
        c, _, _ = mk().step(oracle_mod.make_params(h=h, n_it=8, v_imp=1e30, ordering=o))
        err[o] = np.abs(c["P"][:, 0] - ref["P"][:, 0]).max()
    assert err[1] < 0.5 * err[0]


def test_kinematic_and_force_driven_plate(oracle_mod):
    """A velocity-driven axis advances exactly u h per step; a force-driven plate pressing
    a sphere onto the floor reaches the static balance F_p = -F_applied, floor = F + m g."""
    r, h = 4.25e-3, 1e-4
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    P = oracle_mod.make_plate([(-0.01, -0.01, 0.0)], [(0.01, 0.01, 0.005)], pos=(0.5, 0.5, 0.5), mass=0.05)
    P.mode[0], P.target[0], P.vel[0] = 1, 0.1, 0.1
    W = oracle_mod.OracleWorld([[0, 0, r]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor, plates=[P])
    p = oracle_mod.make_params(h=h, n_it=20, E=1e9, nu=0.15, rho=2200.0)
    x0 = W.plates[0].pos[0]
    for k in range(1, 11):
        W.step(p)
        assert W.plates[0].pos[0] == x0 + sum([h * 0.1] * k) or abs(W.plates[0].pos[0] - (x0 + k * h * 0.1)) < 1e-15
    # force axis
    F0 = 2.0
    P = oracle_mod.make_plate([(-0.01, -0.01, 0.0)], [(0.01, 0.01, 0.005)], pos=(0, 0, 2 * r - 1e-6), mass=0.05)
    P.mode[2], P.target[2] = 2, -F0
    W = oracle_mod.OracleWorld([[0, 0, r]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor, plates=[P])
    p = oracle_mod.make_params(h=h, n_it=50, E=1e9, nu=0.15, rho=2200.0)
    for _ in range(1500):
        c, _, _ = W.step(p)
    m, _ = oracle_mod.mass_inertia(2 * r, 2200.0)
    assert W.plates[0].force[2] == pytest.approx(F0, rel=0.01)
    f = {int(k) & 0xFFFFFFFF: c["P"][i, 0] / h for i, k in enumerate(c["key"])}
    assert f[oracle_mod.WALL_KEY_BASE + 4] == pytest.approx(F0 + m * 9.81, rel=0.01)


def test_motor_force_limits(oracle_mod):
    """Eq. 4 on a plate motor, staggered reading R18: a force-limited velocity axis
    accelerates a free plate at f_max/m (staggered: x_n = x_0 + a h^2 n(n-1)/2) until it reaches
    u, then holds u with zero motor force; a locked plate under a resting sphere carries its weight;
    a press whose motor saturates at f_min reduces to a force axis (static balance F_p = -f_min)."""
    r, h = 4.25e-3, 1e-4
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    p = oracle_mod.make_params(h=h, n_it=20, E=1e9, nu=0.15, rho=2200.0)
    for sgn in (1.0, -1.0):
        u, F, m = 0.1 * sgn, 0.1, 0.05
        a = F / m
        P = oracle_mod.make_plate([(-0.01, -0.01, 0.0)], [(0.01, 0.01, 0.005)], pos=(0.5, 0.5, 0.5), mass=m)
        P.mode[0], P.target[0], P.limit[0] = 1, u, 1
        P.fmin[0], P.fmax[0] = (-math.inf, F) if sgn > 0 else (-F, math.inf)
        W = oracle_mod.OracleWorld([[0, 0, r]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor, plates=[P])
        x0 = W.plates[0].pos[0]
        for n in range(1, 401):
            W.step(p)
            assert W.plates[0].pos[0] - x0 == pytest.approx(sgn * a * h * h * n * (n - 1) / 2, rel=1e-12, abs=2.5e-16 * n)
            assert W.plates[0].motor[0] == sgn * F
        W.step(p, 200)
        assert W.plates[0].vel[0] == u and W.plates[0].motor[0] == 0.0
    # locked plate as the floor under a resting sphere: the motor carries m g (upward)
    P = oracle_mod.make_plate([(-0.01, -0.01, -0.005)], [(0.01, 0.01, 0.0)], pos=(0, 0, 0), mass=0.05)
    W = oracle_mod.OracleWorld([[0, 0, r]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], plates=[P])
    W.step(p, 300)
    mp, _ = oracle_mod.mass_inertia(2 * r, 2200.0)
    assert W.plates[0].force[2] == pytest.approx(-mp * 9.81, rel=0.01)
    assert W.plates[0].motor[2] == pytest.approx(mp * 9.81, rel=0.01)
    # a press at -0.05 m/s limited to f_min = -F0 balances like a force axis of -F0
    F0 = 2.0
    P = oracle_mod.make_plate([(-0.01, -0.01, 0.0)], [(0.01, 0.01, 0.005)], pos=(0, 0, 2 * r - 1e-6), mass=0.05)
    P.mode[2], P.target[2], P.limit[2], P.fmin[2], P.fmax[2] = 1, -0.05, 1, -F0, math.inf
    W = oracle_mod.OracleWorld([[0, 0, r]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor, plates=[P])
    p = oracle_mod.make_params(h=h, n_it=50, E=1e9, nu=0.15, rho=2200.0)
    c, _, _ = W.step(p, 1500)
    assert W.plates[0].motor[2] == -F0
    assert W.plates[0].force[2] == pytest.approx(F0, rel=0.01)
    f = {int(k) & 0xFFFFFFFF: c["P"][i, 0] / h for i, k in enumerate(c["key"])}
    assert f[oracle_mod.WALL_KEY_BASE + 4] == pytest.approx(F0 + mp * 9.81, rel=0.01)


def test_monolithic_plate_coupling(oracle_mod):
    """Reading R18b (SURVEY NEXT-3 'monolithic plate coupling'): a force-driven plate axis as a
    body of the main-stage solve.  Pins: (1) a free plate under a constant force F integrates
    symplectically, x_n = x_0 + a h^2 n(n+1)/2 (the staggered R18 gives n(n-1)/2); (2) pressing
    a sphere onto the floor it reaches the static balance F_p = -F, floor = F + m g; (3) a free
    plate (all axes force-driven, F = 0) striking a free sphere conserves the total momentum to
    rounding at every step (the plate takes exactly the impulses the sphere gives)."""
    r, h = 4.25e-3, 1e-4
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    F, m = 0.2, 0.05
    P = oracle_mod.make_plate([(-0.01, -0.01, 0.0)], [(0.01, 0.01, 0.005)], pos=(0.5, 0.5, 0.5), mass=m)
    P.mode[0], P.target[0] = 2, F
    W = oracle_mod.OracleWorld([[0, 0, r]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor, plates=[P])
    p = oracle_mod.make_params(h=h, n_it=20, E=1e9, nu=0.15, rho=2200.0, plate_coupling=1)
    x0 = W.plates[0].pos[0]
    for n in range(1, 101):
        W.step(p)
        assert W.plates[0].pos[0] - x0 == pytest.approx(F / m * h * h * n * (n + 1) / 2, rel=1e-12, abs=2.5e-16 * n)
    # (2) static press
    F0 = 2.0
    P = oracle_mod.make_plate([(-0.01, -0.01, 0.0)], [(0.01, 0.01, 0.005)], pos=(0, 0, 2 * r - 1e-6), mass=0.05)
    P.mode[2], P.target[2] = 2, -F0
    W = oracle_mod.OracleWorld([[0, 0, r]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor, plates=[P])
    p = oracle_mod.make_params(h=h, n_it=50, E=1e9, nu=0.15, rho=2200.0, plate_coupling=1)
    c, _, _ = W.step(p, 1500)
    mp, _ = oracle_mod.mass_inertia(2 * r, 2200.0)
    assert W.plates[0].force[2] == pytest.approx(F0, rel=0.01)
    f = {int(k) & 0xFFFFFFFF: c["P"][i, 0] / h for i, k in enumerate(c["key"])}
    assert f[oracle_mod.WALL_KEY_BASE + 4] == pytest.approx(F0 + mp * 9.81, rel=0.01)
    # (3) momentum
    P = oracle_mod.make_plate([(-0.01, -0.01, -0.01)], [(0.01, 0.01, 0.01)], pos=(0.05, 0.0, 0.0), mass=0.02)
    for k in range(3):
        P.mode[k], P.target[k] = 2, 0.0
    P.vel[0] = -0.3
    W = oracle_mod.OracleWorld([[0.05 - 0.01 - r - 2e-5, 0.001, -0.002]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0],
                               plates=[P])
    p = oracle_mod.make_params(h=1e-5, n_it=30, E=1e9, nu=0.15, rho=2200.0, g=(0, 0, 0), plate_coupling=1)
    mom0 = 0.02 * np.array(W.plates[0].vel[:])
    hit = False
    for _ in range(60):
        c, _, _ = W.step(p)
        hit = hit or len(c) > 0
        mom = 0.02 * np.array(W.plates[0].vel[:]) + mp * W.v[0]
        assert np.abs(mom - mom0).max() <= 1e-12 * 0.02 * 0.3
    assert hit and W.v[0, 0] < -0.05                                 # the sphere was struck


# ---------------------------------------------------------------- outputs of the step (O6, O9, R19)

def test_forces_torques_k_stack(oracle_mod):
    """O6 per-particle outputs F = (1/h) sum +-(P_n n + P_t), T = (1/h) sum +-(l x P_t + P_r)
    (Eq. 2: the contact forces are G^T lambda).  A settled column of k spheres is in
    equilibrium: every sphere's net contact force balances its weight, F = +m g z (a sign error on
    either body, a dropped 1/h or a missing floor contact fails), and no torque acts (the column
    is symmetric: P_t = 0)."""
    k, r, h = 4, 4.25e-3, 1e-4
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    x = np.array([[0, 0, r + 2 * r * i] for i in range(k)])
    W = oracle_mod.OracleWorld(x, np.zeros((k, 3)), np.zeros((k, 3)), [r] * k, np.arange(k), walls=floor)
    p = oracle_mod.make_params(h=h, n_it=200, E=1e9, nu=0.15, rho=2200.0)
    for _ in range(400):
        W.step(p)
    _, F, T = W.step(p, want_forces=True)
    m, _ = oracle_mod.mass_inertia(2 * r, 2200.0)
    for i in range(k):
        np.testing.assert_allclose(F[i], [0.0, 0.0, m * 9.81], rtol=0, atol=0.01 * m * 9.81)
    assert np.all(T == 0.0)


def test_forces_torques_static_incline(oracle_mod):
    """A sphere held static on a plane under gravity tilted by theta with tan(theta) <= mu_r
    (reading R7: rolling bound mu_r R* P_n, R* = r for a wall).  Equilibrium of the
    free body: the contact force balances gravity, F = -m g; the contact torque vanishes, T = 0;
    so the rolling-resistance moment balances the friction moment about the centre,
    |P_r|/h = |l| m g sin(theta) with the lever arm |l| = r - delta/2 (reading R10, the midpoint of
    the overlap lens).  A soft material makes delta/2r ~ 3 %, so a lever arm of r (or a flipped
    torque sign, or a dropped rolling term) fails."""
    mu_t, mu_r, r, h = 0.4, 0.1, 3e-3, 1e-4
    E, nu = 1e5, 0.3
    th = math.atan(0.08)
    g = 9.81
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4, mu_t=mu_t, mu_r=mu_r)
    m, _ = oracle_mod.mass_inertia(2 * r, RHO)
    kn = (E / (2 * (1 - nu * nu))) * math.sqrt(2 * r) / 3
    d0 = (m * g * math.cos(th) / kn) ** (2 / 3)
    assert d0 / (2 * r) > 0.02
    W = oracle_mod.OracleWorld([[0, 0, r - d0]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor)
    gv = np.array([g * math.sin(th), 0.0, -g * math.cos(th)])
    p = oracle_mod.make_params(h=h, n_it=100, E=E, nu=nu, mu_t=mu_t, mu_r=mu_r, g=tuple(gv))
    for _ in range(4000):
        W.step(p)
    c, F, T = W.step(p, want_forces=True)
    assert abs(W.v[0]).max() < 1e-7 and abs(W.w[0]).max() < 1e-4
    np.testing.assert_allclose(F[0], -m * gv, rtol=0, atol=1e-4 * m * g)
    lever = r - c["delta"][0] / 2
    M = lever * m * g * math.sin(th)
    assert np.abs(T[0]).max() < 1e-4 * M
    assert np.linalg.norm(c["P"][0, 4:7]) / h == pytest.approx(M, rel=2e-4)
    assert abs(np.linalg.norm(c["P"][0, 4:7]) / h - r * m * g * math.sin(th)) > 0.01 * M   # not r


def test_residual_report_closed_forms(oracle_mod):
    """O9 report: max |min(P_n, u_n + Sigma P_n - b)| at the final velocities.
    (a) One normal row is solved exactly by one Jacobi sweep (c = 1: the split diagonal is the
    true one), so its residual is 0.  (b) Two spheres stacked on a floor, frictionless, one sweep
    from P = 0: with mass splitting the lower sphere has c = 2, so D_1 = 2/m, D_2 = 3/m; writing
    u_c - b_c = -(D_c + S_c) P_c and the velocity changes (P_1 - P_2)/m, P_2/m, both rows end at
    u' + S P - b = -(P_1 + P_2)/m: the residual is (P_1 + P_2)/m (no mass splitting would give
    max(P_1, P_2)/m)."""
    r, h = 4.25e-3, 1e-4
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    p = oracle_mod.make_params(h=h, n_it=1, E=1e9, nu=0.15, rho=2200.0, mu_t=0.0, mu_r=0.0, g=(0, 0, 0),
                               v_imp=1e30)
    m, _ = oracle_mod.mass_inertia(2 * r, 2200.0)
    # (a) one sphere pressed 1 um into the floor, approaching at 1 mm/s
    W = oracle_mod.OracleWorld([[0, 0, r - 1e-6]], [[0, 0, -1e-3]], np.zeros((1, 3)), [r], [0], walls=floor)
    c, _, _ = W.step(p)
    assert len(c) == 1 and c["P"][0, 0] > 0
    assert W.last_report.max_normal_residual <= 1e-12 * (1e-3 + c["P"][0, 0] / m)
    # (b) two-sphere stack, both contacts compressed
    x = np.array([[0, 0, r - 1e-6], [0, 0, 3 * r - 3e-6]])
    W = oracle_mod.OracleWorld(x, np.zeros((2, 3)), np.zeros((2, 3)), [r, r], [0, 1], walls=floor)
    c, _, _ = W.step(p)
    assert len(c) == 2 and np.all(c["P"][:, 0] > 0)
    P1, P2 = c["P"][:, 0]
    res = W.last_report.max_normal_residual
    assert res == pytest.approx((P1 + P2) / m, rel=1e-9)
    assert abs(res - max(P1, P2) / m) > 0.1 * res
    # (c) the report's cone excess max(|P_t| - mu_t P_n, |P_r| - mu_r R* P_n, 0): a sphere sliding
    # down a steep incline sits on the friction cone (|P_t| = mu_t P_n), so the
    # excess is zero to rounding while |P_t| is at the limit
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4, mu_t=0.4, mu_r=0.1)
    th = math.atan(1.4)
    W = oracle_mod.OracleWorld([[0, 0, r]], np.zeros((1, 3)), np.zeros((1, 3)), [r], [0], walls=floor)
    pp = oracle_mod.make_params(h=h, n_it=60, E=1e9, nu=0.15, rho=2200.0, g=(9.81 * math.sin(th), 0, -9.81 * math.cos(th)))
    for _ in range(200):
        c, _, _ = W.step(pp)
    assert np.linalg.norm(c["P"][0, 1:4]) == pytest.approx(0.4 * c["P"][0, 0], rel=1e-9)
    assert 0.0 <= W.last_report.max_cone_excess <= 1e-12 * c["P"][0, 0]


def test_centre_inside_plate_box_dense_directions(oracle_mod):
    """Reading R19 (PAPER silent): a sphere whose centre lies inside a grouser box is pushed out
    along the shortest way.  Brute force: over a dense set of directions d, the smallest
    translation t(d) after which the sphere no longer touches the box (distance from the box
    >= r, found by bisection) is the overlap delta, and the minimising d is -n (n points from the
    particle into the box)."""
    lo, hi = np.array([0.0, 0.0, 0.0]), np.array([0.0255, 0.05, 0.043])
    P = oracle_mod.make_plate([lo], [hi], pos=(0, 0, 0), mass=1.0)
    r = 3e-3
    ng = 40000
    i = np.arange(ng) + 0.5
    phi = np.arccos(1 - 2 * i / ng)
    th = np.pi * (1 + 5 ** 0.5) * i
    D = np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], 1)

    def box_dist(Y):
        q = np.clip(Y, lo, hi)
        return np.linalg.norm(Y - q, axis=-1)

    for X in [np.array([0.004, 0.03, 0.02]), np.array([0.02, 0.0475, 0.01]), np.array([0.012, 0.02, 0.0415])]:
        c, _ = _world(oracle_mod, [X], [r], plates=[P]).detect()
        assert len(c) == 1
        a, b = np.zeros(ng), np.full(ng, 0.2)
        for _ in range(60):
            mid = 0.5 * (a + b)
            out = box_dist(X + mid[:, None] * D) >= r
            b = np.where(out, mid, b)
            a = np.where(out, a, mid)
        k = np.argmin(b)
        assert c["delta"][0] == pytest.approx(b[k], rel=1e-3)
        np.testing.assert_allclose(c["n"][0], -D[k], atol=0.02)
        depth = min((X - lo).min(), (hi - X).min())
        assert c["delta"][0] > r + 0.9 * depth


def test_openmp_sweeps_bit_identical(oracle_mod):
    """OpenMP over contacts and particles is allowed because Jacobi is order-free;
    the oracle solves each contact alone and sums each body's increments in contact order, so
    any thread count gives the same bits (5 steps of an 8x polydisperse cloud with walls)."""
    import synth
    b = synth.random_cloud(1500, (0, 0, 0), (0.06, 0.06, 0.06), 1e-3, 5e-3, 3, v_scale=0.05, w_scale=2.0,
                           loguniform=True)
    out = []
    n0 = oracle_mod.set_threads(0)
    try:
        for nt in (1, 4):
            oracle_mod.set_threads(nt)
            W = oracle_mod.OracleWorld(b.x, b.v, b.w, b.r, b.gid,
                                       walls=oracle_mod.box_walls(b.box_lo, b.box_hi, mu_t=0.2, mu_r=0.05))
            c, F, T = W.step(oracle_mod.make_params(h=1e-5, n_it=40), 5, want_forces=True)
            out.append((W.x.copy(), W.v.copy(), W.w.copy(), c["P"].copy(), F, T))
    finally:
        oracle_mod.set_threads(n0)
    for u, v in zip(*out):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("n_it", [1, 2, 7])
def test_mass_splitting_duplicated_support_is_exact(oracle_mod, n_it):
    """The finite-N_it Jacobi iterate with mass splitting (reading C22: contact j of
    body i sees the inverse mass c_i/m_i, the body update sums the increments with 1/m_i).  A
    sphere resting on TWO coincident frictionless floors (c = 2) has duplicated normal rows; the
    exact LCP gives each half of Lambda = -(u + b)/(1/m + Sigma/2), and the mass-split Jacobi
    reaches it after ONE sweep and stays there (each copy solves -(u + b)/(2/m + Sigma)).  SPOOK's
    bias b does not depend on the stiffness and Sigma ~ 1/k, so the result equals a
    single floor of doubled stiffness solved exactly (one row: one sweep).  A split count of 1
    (or an update scaled by c/m) overshoots by ~2x; an average instead of a sum undershoots."""
    r, h, k, d0, rho = 5e-3, 1e-4, 2e4, 2e-5, 2600.0
    floor = oracle_mod.box_walls((-1, -1, 0), (1, 1, 1), mask=1 << 4)
    out = {}
    for tag, walls, kl in (("dup", list(floor) * 2, k), ("one2k", list(floor), 2 * k), ("onek", list(floor), k)):
        W = oracle_mod.OracleWorld([[0, 0, r - d0]], [[0.0, 0.0, -0.01]], np.zeros((1, 3)), [r], [0], walls=walls)
        c, _, _ = W.step(oracle_mod.make_params(h=h, n_it=n_it, e_H=1.0, k_lin=kl, rho=rho))
        assert len(c) == len(walls) and W.last_report.impact_fired == 0
        out[tag] = (W.v[0].copy(), W.x[0].copy(), c["P"][:, 0].sum())
    vd, xd, Pd = out["dup"]
    v2, x2, P2 = out["one2k"]
    assert vd[2] == pytest.approx(v2[2], rel=1e-12, abs=1e-15)
    assert xd[2] == pytest.approx(x2[2], rel=1e-14)
    assert Pd == pytest.approx(P2, rel=1e-12)
    assert abs(out["onek"][2] - P2) > 1e-3 * abs(P2)           # the stiffness matters at this size
