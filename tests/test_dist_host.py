"""Host logic of the x-slab decomposition with world_size 2 over
gloo on the CPU: the per-rank slab inputs bench.py builds, the slab faces, and the ghost-band
rule the library applies (band width W = 2 r_max + 2 skin, include/dem.h), checked against a
brute-force neighbour search of the assembled bed: every pair within r_a + r_b + skin that has
one particle owned by a rank has the other one in that rank's owned set or ghost band."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _piece(rank):
    b = synth.banded_bed((0.06, 0.03, 0.03), [(0.0, 0.01, 1e-3), (0.01, 0.03, 2e-3)], 77 + rank, spacing=2.0)
    return synth.shift_slab(b, rank, WORLD)


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        bed, slab = _piece(rank)
        # faces agree: my hi is my right neighbour's lo
        faces = [None] * WORLD
        dist.all_gather_object(faces, slab)
        ok_faces = all(faces[r][1] == faces[r + 1][0] for r in range(WORLD - 1))
        inside = bool(np.all((bed.x[:, 0] >= slab[0]) & (bed.x[:, 0] < slab[1])))
        # the assembled bed
        parts = [None] * WORLD
        dist.all_gather_object(parts, (bed.x, bed.r, bed.gid))
        x = np.concatenate([p[0] for p in parts])
        r = np.concatenate([p[1] for p in parts])
        # particles move after the start: a seeded x-shuffle of up to 3 mm makes pairs straddle the
        # face; ownership is by position, as the library assigns it at every rebuild
        x = x.copy()
        x[:, 0] += np.random.default_rng(5).uniform(-3e-3, 3e-3, len(x))
        gid = np.concatenate([p[2] for p in parts])
        unique = len(np.unique(gid)) == len(gid)
        # ghost band rule of the library: skin = 0.1 r_min (default), W = 2 r_max + 2 skin
        skin = 0.1 * r.min()
        W = 2.0 * r.max() + 2.0 * skin
        owned = ((x[:, 0] >= slab[0]) | (rank == 0)) & ((x[:, 0] < slab[1]) | (rank == WORLD - 1))   # outer slabs open
        ghost = ~owned & (((x[:, 0] >= slab[0] - W) & (x[:, 0] < slab[0]) & (rank > 0)) |
                          ((x[:, 0] >= slab[1]) & (x[:, 0] < slab[1] + W) & (rank < WORLD - 1)))
        local = owned | ghost
        from scipy.spatial import cKDTree
        pairs = cKDTree(x).query_pairs(2 * r.max() + skin, output_type="ndarray")
        d = np.linalg.norm(x[pairs[:, 0]] - x[pairs[:, 1]], axis=1)
        pairs = pairs[d < r[pairs[:, 0]] + r[pairs[:, 1]] + skin]
        touch = owned[pairs[:, 0]] | owned[pairs[:, 1]]
        covered = bool(np.all(local[pairs[touch, 0]] & local[pairs[touch, 1]]))
        cross = int(np.sum(owned[pairs[:, 0]] != owned[pairs[:, 1]]))
        q.put((rank, ok_faces, inside, unique, covered, cross, int(owned.sum()), int(ghost.sum())))
    finally:
        dist.destroy_process_group()


def test_slab_pieces_and_ghost_band_cover_every_cross_face_pair():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in ps:
        p.start()
    out = [q.get(timeout=240) for _ in range(WORLD)]
    for p in ps:
        p.join(timeout=60)
    out.sort()
    n_total = sum(o[6] for o in out)
    for rank, ok_faces, inside, unique, covered, cross, n_own, n_ghost in out:
        assert ok_faces and inside and unique, out
        assert covered, f"rank {rank}: a pair touching an owned particle is missing from the local set"
        assert n_ghost > 0
    assert out[0][5] > 0                                  # pairs straddle the face: the exchange is real
    assert n_total == sum(_piece(r)[0].n for r in range(WORLD))   # every particle owned once


def test_slab_bounds_helper_quantiles():
    from paper_2501_05300_b200 import dem
    x = np.linspace(0.0, 1.0, 1001)
    b = dem.slab_bounds(x, 4, 0.0, 1.0)
    assert b[0] == 0.0 and b[-1] == 1.0 and len(b) == 5
    counts = [np.sum((x >= b[i]) & (x < b[i + 1])) for i in range(4)]
    assert max(counts) - min(counts) <= 2
