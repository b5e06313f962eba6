"""On-device bed generator (include/dem.h dem_generator): the particles it creates on
the GPU, single context and split over loopback ranks (x-slab decomposition)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BANDS = [(0.02, 1e-3), (0.05, 2e-3)]                          # fine over coarse (config 1 shape)
BOX = dict(lo=(0.0, 0.0, 0.0), hi=(0.06, 0.04, 0.05))


def dem():
    from paper_2501_05300_b200 import dem as D
    return D


def test_generated_bed_properties_and_determinism():
    from scipy.spatial import cKDTree
    D = dem()
    gen = dict(kind="bands", bands=BANDS, spacing_factor=2.25, seed=42)
    b = D.Bed(generator=gen, box=BOX, solver=dict(dt=1e-5, n_iter=10))
    st = b.get_state()
    b.close()
    n = D.generator_count(gen, BOX)
    assert len(st["gid"]) == n and np.array_equal(st["gid"], np.arange(n, dtype=np.uint32))
    r, x = st["radius"], st["pos"]
    fine = x[:, 2] > BOX["hi"][2] - 0.02
    assert np.all((r[fine] >= 0.9e-3 - 1e-15) & (r[fine] <= 1.1e-3 + 1e-15))
    assert np.all((r[~fine] >= 1.8e-3 - 1e-15) & (r[~fine] <= 2.2e-3 + 1e-15))
    assert r[fine].std() > 0.03e-3                             # the +-10 % jitter is there
    # sites sit 1.1 r_nom from the walls; radius (<= 1.1 r_nom) plus jitter (0.01 r_nom) may touch them
    tol = (0.0111 * r / 0.9)[:, None]
    assert np.all(x - r[:, None] >= np.array(BOX["lo"]) - tol) and np.all(x + r[:, None] <= np.array(BOX["hi"]) + tol)
    pairs = cKDTree(x).query_pairs(2 * r.max(), output_type="ndarray")
    d = np.linalg.norm(x[pairs[:, 0]] - x[pairs[:, 1]], axis=1)
    assert np.all(d > r[pairs[:, 0]] + r[pairs[:, 1]])       # spacing 2.25: nobody touches at t = 0
    assert np.all(st["vel"] == 0.0)
    b2 = D.Bed(generator=gen, box=BOX, solver=dict(dt=1e-5, n_iter=10))
    st2 = b2.get_state()
    b2.close()
    assert np.array_equal(st2["pos"], st["pos"]) and np.array_equal(st2["radius"], st["radius"])
    b3 = D.Bed(generator=dict(gen, seed=43), box=BOX, solver=dict(dt=1e-5, n_iter=10))
    assert not np.array_equal(b3.get_state()["pos"], st["pos"])
    b3.close()


@pytest.mark.parametrize("kind", ["profile", "layers"])
def test_generated_graded_beds_grow_with_depth(kind):
    D = dem()
    gen = dict(kind=kind, d_min=2e-3, gamma=0.1, d_max=6e-3, ratio_r=1.5, eta=3.0, seed=7)
    box = dict(lo=(0.0, 0.0, 0.0), hi=(0.05, 0.03, 0.08))
    b = D.Bed(generator=gen, box=box, solver=dict(dt=1e-5, n_iter=10))
    st = b.get_state()
    b.close()
    depth = box["hi"][2] - st["pos"][:, 2]
    top, bottom = st["radius"][depth < 0.01].mean(), st["radius"][depth > 0.06].mean()
    assert len(st["gid"]) == D.generator_count(gen, box)
    assert bottom > 1.5 * top                                  # radius grows with depth


def test_generated_slabs_over_loopback_ranks_union_to_the_bed():
    """Each rank generates the sites of its slab under their global gids: the union of the ranks'
    owned particles after the first rebuild is the single-rank bed, particle for particle."""
    import threading
    D = dem()
    gen = dict(kind="bands", bands=BANDS, spacing_factor=2.0, seed=9)
    one = D.Bed(generator=gen, box=BOX, solver=dict(dt=1e-5, n_iter=10))
    ref = one.get_state()
    one.close()
    G, faces = 3, [0.0, 0.021, 0.04, 0.06]
    grp = D.LoopbackGroup(G)
    out, err = [None] * G, [None] * G

    def rank(r):
        try:
            b = D.Bed(generator=gen, box=BOX, solver=dict(dt=1e-5, n_iter=10),
                      dist=dict(rank=r, world_size=G, slab=(faces[r], faces[r + 1]), transport="loopback", group=grp))
            b.step(2)
            out[r] = (b.get_state(), b.n_owned)
            b.close()
        except Exception as e:   # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=rank, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    grp.close()
    for e in err:
        if e is not None:
            raise e
    gids = np.concatenate([o[0]["gid"] for o in out])
    assert len(gids) == len(ref["gid"]) and np.array_equal(np.sort(gids), ref["gid"])
    assert all(o[1] > 0 for o in out)
    r0 = np.concatenate([o[0]["radius"] for o in out])[np.argsort(gids)]
    assert np.array_equal(r0, ref["radius"])
