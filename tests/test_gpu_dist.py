"""x-slab domain decomposition on one GPU: G loopback ranks in one
process (include/dem.h dem_loopback_create) against a single context on the whole bed.

The ranks own disjoint slabs, hold ghost bands of their neighbours, exchange ghost velocities
after every Jacobi sweep and re-assign ownership at every rebuild.  Every contact is evaluated in
its canonical orientation (body a = smaller gid), each particle's half-contacts are ordered by
partner gid and summed by the same scan tree whatever warp holds them, and plate reactions are
int64 sums: the decomposed run reproduces the single context BIT FOR BIT,
whatever the number of slabs and wherever the faces fall.
"""
import numpy as np
import pytest

import synth
from tests.parity import run_loopback

pytestmark = pytest.mark.gpu


def dem():
    from paper_2501_05300_b200 import dem as D
    return D


def single(bed, n_steps, solver, box, plates=()):
    b = dem().Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=solver, box=box)
    pids = [b.add_plate(**p) for p in plates]
    reps = [b.step(1) for _ in range(n_steps)]
    out = dict(state=b.get_state(), contacts=b.get_contacts(), forces=b.get_forces(), reports=reps,
               plates=[b.get_plate(p) for p in pids],
               walls=[b.get_wall(w) for w in range(6) if (box.get("wall_mask", 0x3F) >> w) & 1])
    b.close()
    return out


def drifting_bed(drift=5.0, seed=11):
    """A jammed polydisperse lattice (overlaps relax smoothly, impacts fire) drifting along x with
    no x-walls: particles cross the slab faces, so rebuilds move ownership between ranks.  The
    drift leaves relative motion unchanged, and the bed is not chaotic over these steps, so the
    decomposed run can be held to the single context at rounding level."""
    bed = synth.banded_bed((0.12, 0.04, 0.04), [(0.0, 0.04, 2e-3)], seed, spacing=2.05)
    bed.v[:, 0] = drift
    return bed, dict(lo=(0.0, 0.0, 0.0), hi=(0.12, 0.04, 0.04), wall_mask=0x3C)


@pytest.mark.parametrize("G", [2, 3])
def test_loopback_matches_single_context(G):
    bed, box = drifting_bed()
    solver = dict(dt=2e-5, n_iter=30)
    n_steps = 12
    ref = single(bed, n_steps, solver, box)
    # faces 0.3 mm ahead of a lattice plane: the drifting plane crosses within a few steps
    xs = np.unique(np.round(bed.x[:, 0], 4))
    faces = [float(xs[np.searchsorted(xs, 0.12 * k / G)]) + 3e-4 for k in range(1, G)]
    out = run_loopback(bed, G, n_steps, solver, box, bounds=[0.0] + faces + [0.12])
    st, rs = out["state"], ref["state"]
    assert np.array_equal(st["gid"], rs["gid"])                      # every particle owned exactly once
    for k in ("pos", "vel", "angvel"):                               # bit-identical trajectories
        assert np.array_equal(st[k], rs[k]), k
    assert np.array_equal(out["contacts"]["key"], ref["contacts"]["key"])   # pair set, each contact once
    assert np.array_equal(out["contacts"]["P"], ref["contacts"]["P"])
    assert np.array_equal(out["contacts"]["n"], ref["contacts"]["n"])
    # global step reports: contacts and impact decisions identical on every rank
    for r in out["ranks"]:
        for a, b in zip(r["reports"], ref["reports"]):
            assert a["n_contacts"] == b["n_contacts"] and a["impact_fired"] == b["impact_fired"]
            assert a["rebuilt"] == b["rebuilt"]
            assert abs(a["ke"] - b["ke"]) <= 1e-9 * max(b["ke"], 1e-30)
    # the bed drifted across the faces: rebuilds moved ownership between the ranks
    assert any(rep["rebuilt"] for rep in ref["reports"][1:])
    assert any(r["n_owned"] != int(((bed.x[:, 0] >= out["bounds"][k]) & (bed.x[:, 0] < out["bounds"][k + 1])).sum())
               for k, r in enumerate(out["ranks"]))


def test_loopback_plate_reaction_summed_over_ranks():
    """A force-driven plate spanning both slabs: its reaction is the int64 sum over the ranks
    of their owned contacts, identical on every rank and equal to the single context's."""
    bed, box = drifting_bed(drift=0.0, seed=5)
    top = float((bed.x[:, 2] + bed.r).max())
    plate = dict(boxes_lo=[(-0.05, -0.015, 0.0)], boxes_hi=[(0.05, 0.015, 0.004)], pos=(0.06, 0.02, top - 0.0005),
                 mass=0.5)
    solver = dict(dt=2e-5, n_iter=30, gravity=(0.0, 0.0, -9.81))
    ref = single(bed, 8, solver, box, plates=[plate])
    out = run_loopback(bed, 2, 8, solver, box, plates=[plate])
    f_ref = np.array(ref["plates"][0]["force"])
    assert ref["plates"][0]["n_contacts"] > 0
    for r in out["ranks"]:
        p = r["plates"][0]
        assert p["n_contacts"] == ref["plates"][0]["n_contacts"]
        assert np.array_equal(np.array(p["force"]), f_ref)
        assert p["pos"] == ref["plates"][0]["pos"]
    for k in ("pos", "vel", "angvel"):
        assert np.array_equal(out["state"][k], ref["state"][k]), k


@pytest.mark.parametrize("transport", ["nccl", "nccl_graph", "loopback"])
def test_single_rank_transport_selftest_bit_identical(transport, monkeypatch):
    """world_size 1 over a real transport (NCCL communicator of one rank, or a loopback group of
    one) runs the decomposed code path -- ownership pass, band exchange with no neighbours,
    allreduces -- and must reproduce the undecomposed context bit for bit.  nccl_graph: the
    decomposed sweep loop (sweeps, halo pack, grouped NCCL send/recv, unpack) captured in a CUDA
    graph (DEM_GRAPH_NCCL=1)."""
    D = dem()
    if transport == "nccl_graph":
        monkeypatch.setenv("DEM_GRAPH_NCCL", "1")
        transport = "nccl"
    bed, box = drifting_bed(drift=1.0, seed=7)
    solver = dict(dt=2e-5, n_iter=20)
    ref = single(bed, 6, solver, box)
    grp = D.LoopbackGroup(1) if transport == "loopback" else None
    cfg = dict(rank=0, world_size=1, slab=(0.0, 0.12), transport=transport)
    if grp:
        cfg["group"] = grp
    else:
        cfg["nccl_id"] = D.nccl_unique_id()
    b = D.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=solver, box=box, dist=cfg)
    reps = [b.step(1) for _ in range(6)]
    st = b.get_state()
    b.close()
    if grp:
        grp.close()
    for k in ("pos", "vel", "angvel"):
        assert np.array_equal(st[k], ref["state"][k]), k
    assert [r["n_contacts"] for r in reps] == [r["n_contacts"] for r in ref["reports"]]


@pytest.mark.parametrize("G", [2, 4])
def test_chaotic_bed_bit_identical_across_slab_counts(G):
    """A falling polydisperse cloud (impacts, rebuilds, walls, a force-driven plate, 80 steps) is
    chaotic: any rounding difference would grow visibly.  1 context vs G loopback slabs with
    irregular faces: states, contacts, per-particle forces and the plate bit-identical."""
    bed = synth.random_cloud(800, (0.002, 0.002, 0.002), (0.118, 0.038, 0.03), 1.5e-3, 3.0e-3, 3, v_scale=0.3)
    box = dict(lo=(0.0, 0.0, 0.0), hi=(0.12, 0.04, 0.06), wall_mask=0x3F)
    plate = dict(boxes_lo=[(-0.02, -0.01, 0.0)], boxes_hi=[(0.02, 0.01, 0.003)], pos=(0.061, 0.02, 0.02),
                 mass=0.05)
    solver = dict(dt=2e-5, n_iter=25)
    ref = single(bed, 80, solver, box, plates=[plate])
    # irregular faces, interior slabs wider than the ghost band (2 r_max + 2 skin ~ 6.6 mm)
    faces = {2: [0.0437], 4: [0.0231, 0.0517, 0.0893]}[G]
    out = run_loopback(bed, G, 80, solver, box, bounds=[0.0] + list(faces) + [0.12], plates=[plate])
    for k in ("gid", "pos", "vel", "angvel"):
        assert np.array_equal(out["state"][k], ref["state"][k]), k
    assert np.array_equal(out["contacts"]["key"], ref["contacts"]["key"])
    assert np.array_equal(out["contacts"]["P"], ref["contacts"]["P"])
    assert np.array_equal(out["forces"][0], ref["forces"][0]) and np.array_equal(out["forces"][1], ref["forces"][1])
    for r in out["ranks"]:
        assert r["plates"][0]["pos"] == ref["plates"][0]["pos"]
        assert r["plates"][0]["force"] == ref["plates"][0]["force"]
        assert r["walls"] == ref["walls"]                              # wall reactions: int64 sums
    assert any(rep["impact_fired"] for rep in ref["reports"])
    assert any(rep["rebuilt"] for rep in ref["reports"][1:])


def test_thin_interior_slab_rejected_on_every_rank():
    """Ghosts come from the two neighbouring slabs: an interior slab thinner than the ghost band
    is an invalid decomposition, reported by every rank's create (collectively, no hang)."""
    bed, box = drifting_bed(drift=0.0)
    with pytest.raises(Exception) as ei:
        run_loopback(bed, 3, 1, dict(dt=2e-5, n_iter=5), box, bounds=[0.0, 0.06, 0.062, 0.12])
    assert "thinner than the ghost band" in str(ei.value)


def test_reduction_option_is_bit_identical():
    """solver.reduction is kept for the ABI only: the sweep's per-particle sums are exact int64
    fixed point (sweep.cu), so 0 and 1 give the same bits, run to run and across slabs."""
    bed, box = drifting_bed()
    ref = single(bed, 12, dict(dt=2e-5, n_iter=30, reduction=0), box)
    again = single(bed, 12, dict(dt=2e-5, n_iter=30, reduction=1), box)
    for k in ("pos", "vel", "angvel"):
        assert np.array_equal(ref["state"][k], again["state"][k]), k
    out = run_loopback(bed, 2, 12, dict(dt=2e-5, n_iter=30, reduction=1), box)
    for k in ("pos", "vel", "angvel"):
        assert np.array_equal(out["state"][k], ref["state"][k]), k
    assert np.array_equal(out["contacts"]["key"], ref["contacts"]["key"])


def test_rebalance_moves_faces_to_quantiles_bit_identically():
    """dem_rebalance: from a lopsided split (rank 2 owns 2/3 of the bed) the
    faces walk toward the particle-count quantiles, at most one skin per call (a migrating
    particle's contacts and their history are then already on its new owner), and the
    trajectory stays bit-identical to the single context."""
    bed, box = drifting_bed(drift=0.0, seed=9)
    solver = dict(dt=2e-5, n_iter=20)
    n_steps = 60
    ref = single(bed, n_steps, solver, box)
    out = run_loopback(bed, 3, n_steps, solver, box, bounds=[0.0, 0.02, 0.04, 0.12], rebalance_every=1)
    for k in ("gid", "pos", "vel", "angvel"):
        assert np.array_equal(out["state"][k], ref["state"][k]), k
    first = [r["owned"][0] for r in out["ranks"]]
    last = [r["owned"][-1] for r in out["ranks"]]
    assert sum(first) == sum(last) == len(bed.r)
    print("owned first", first, "last", last, "faces", out["ranks"][0]["faces"][-1])
    assert max(first) / min(first) > 3
    assert max(last) < max(first) and min(last) > min(first)            # moving toward balance
    f = [r["faces"] for r in out["ranks"]]
    assert all(fi == f[0] for fi in f)                                  # every rank agrees
    F = np.array(f[0])
    assert np.all(np.diff(F, axis=0) >= 0)                               # monotone toward the quantiles
    assert np.abs(np.diff(F, axis=0)).max() <= 0.1 * bed.r.min() * (1 + 1e-9)   # one skin per call


@pytest.mark.parametrize("drift,G", [(5.0, 2), (-5.0, 3)])
def test_long_drift_hands_over_contact_history(drift, G):
    """The bed drifts 10 mm (two and a half lattice planes) through the faces over 100 steps:
    contacts that formed on one rank enter the neighbour's ghost band and particles change owner
    with their contacts' impulse history (handed over at the rebuilds).  Bit-identical to the
    single context."""
    bed, box = drifting_bed(drift=drift)
    solver = dict(dt=2e-5, n_iter=30)
    ref = single(bed, 100, solver, box)
    out = run_loopback(bed, G, 100, solver, box, bounds=[0.0] + [0.12 * k / G + 3e-4 for k in range(1, G)] + [0.12])
    for k in ("gid", "pos", "vel", "angvel"):
        assert np.array_equal(out["state"][k], ref["state"][k]), k
    assert np.array_equal(out["contacts"]["P"], ref["contacts"]["P"])


def test_long_list_particle_on_a_face_bit_identical():
    """A 12 mm sphere with > 100 contacts straddling a slab face (its list is packed in pieces on
    its owner and its contacts are evaluated on both ranks): bit-identical to one context."""
    from tests.test_gpu_parity import _big_sphere_bed
    bed = _big_sphere_bed()
    box = dict(lo=(0.0, 0.0, 0.0), hi=(0.06, 0.06, 0.06), wall_mask=0x3F)
    solver = dict(dt=1e-5, n_iter=40)
    ref = single(bed, 10, solver, box)
    out = run_loopback(bed, 2, 10, solver, box, bounds=[0.0, 0.0301, 0.06])
    for k in ("gid", "pos", "vel", "angvel"):
        assert np.array_equal(out["state"][k], ref["state"][k]), k


def test_monolithic_plate_across_slabs_bit_identical():
    """R18b with a decomposition: the per-sweep plate impulse sums are exact int64 sums over the
    ranks, so a force-driven plate spanning both slabs moves bit-identically to one context."""
    bed, box = drifting_bed(drift=0.0, seed=5)
    top = float((bed.x[:, 2] + bed.r).max())
    plate = dict(boxes_lo=[(-0.05, -0.015, 0.0)], boxes_hi=[(0.05, 0.015, 0.004)], pos=(0.06, 0.02, top - 0.0005),
                 mass=0.5)
    solver = dict(dt=2e-5, n_iter=30, gravity=(0.0, 0.0, -9.81), plate_coupling=1)

    def run_single():
        D = dem()
        b = D.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=solver, box=box)
        pid = b.add_plate(**plate)
        b.drive_plate(pid, 2, D.AXIS_FORCE, -2.0)
        for _ in range(10):
            b.step(1)
        out = dict(state=b.get_state(), plate=b.get_plate(pid))
        b.close()
        return out
    ref = run_single()
    from tests.parity import run_loopback_driven
    out = run_loopback_driven(bed, 2, 10, solver, box, plate, axis=2, mode=2, target=-2.0)
    for k in ("pos", "vel", "angvel"):
        assert np.array_equal(out["state"][k], ref["state"][k]), k
    for r in out["ranks"]:
        assert r["plate"]["pos"] == ref["plate"]["pos"] and r["plate"]["vel"] == ref["plate"]["vel"]
