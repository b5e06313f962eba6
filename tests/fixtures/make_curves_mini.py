"""Oracle side of the SURVEY §8(d) mini-bed plate curves (tests/curves_mini.py): for each kind
(c1-mini, c2-mini) and seed, settle the bed in the fp64 ORACLE, run the plate protocol for the
full 4e4 / 5e4 steps, and write the plate curve (reaction along the curve axis and the plate
position, per step) to tests/golden/curves_mini_<kind>_<seed>.npz with a digest of the settled
state (the GPU test re-settles with the same oracle and checks the digest).  Produced only by
oracle/ code; run once on the CPU (OpenMP sweeps):
    python tests/fixtures/make_curves_mini.py [kind] [seed]
and the settled beds the GPU test starts from (tests/golden/curves_mini_<kind>_<seed>_settled.npz):
    python tests/fixtures/make_curves_mini.py [kind] [seed] --settled-only
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from tests import curves_mini as CM  # noqa: E402


def settled_path(kind, seed):
    return os.path.join(ROOT, "tests", "golden", f"curves_mini_{kind}_{seed}_settled.npz")


def settled(kind, seed, use_cache=True):
    """the bed settled under gravity by the oracle (cell-list mode), with its contact history.
    The settled state is cached under tests/golden (written by this script from the oracle, see
    save_settled) so that the GPU test does not re-run the oracle's settling on the GPU box; the
    test checks its digest against the one stored with the oracle curve."""
    b = CM.make_bed(kind, seed)
    path = settled_path(kind, seed)
    if use_cache and os.path.exists(path):
        z = np.load(path)
        W = O.OracleWorld(z["x"], z["v"], z["w"], z["r"], z["gid"],
                          walls=O.box_walls(b.box_lo, b.box_hi, mask=CM.WALL_MASK), time=float(z["time"]))
        W.hist = z["hist"].astype(O.CONTACT_DTYPE)
        return b, W
    O.set_binning(True)
    W = O.OracleWorld(b.x, b.v, b.w, b.r, b.gid, walls=O.box_walls(b.box_lo, b.box_hi, mask=CM.WALL_MASK))
    W.step(O.make_params(h=CM.SETTLE["h"], n_it=CM.SETTLE["n_it"]), CM.SETTLE["steps"])
    return b, W


def save_settled(kind, seed):
    """settle with the oracle (never from the cache) and store the state with its digest"""
    b, W = settled(kind, seed, use_cache=False)
    np.savez_compressed(settled_path(kind, seed), x=W.x, v=W.v, w=W.w, r=W.r, gid=W.gid, hist=W.hist,
                        time=W.time, digest=digest(W))
    print("wrote", settled_path(kind, seed), digest(W), flush=True)


def digest(W):
    h = hashlib.sha256()
    for a in (W.x, W.v, W.w, W.hist["key"], W.hist["P"]):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run(kind, seed):
    t0 = time.time()
    b, W = settled(kind, seed)
    dg = digest(W)
    lo, hi, pos, mass, drives = CM.plate(kind, W.x, W.r, b.box_hi)
    P = O.make_plate(lo, hi, pos=pos, mass=mass)
    for ax, mode, target, ramp in drives:
        P.mode[ax], P.target[ax], P.ramp[ax] = mode, target, ramp
        if mode == 1 and ramp == 0.0:
            P.vel[ax] = target
    W.plates = (O.Plate * 1)(P)
    W.n_plates = 1
    W.time = 0.0
    p = O.make_params(h=CM.DT, n_it=CM.N_IT, plate_coupling=CM.plate_coupling(kind))
    ax = CM.curve_axis(kind)
    n = CM.N_STEPS[kind]
    f = np.empty(n)
    x = np.empty(n)
    nc = np.empty(n, dtype=np.int32)
    t1 = time.time()
    for s in range(n):
        c, _, _ = W.step(p)
        f[s] = W.plates[0].force[ax]
        x[s] = W.plates[0].pos[ax]
        nc[s] = W.last_report.n_plate
        if s % 5000 == 0:
            print(kind, seed, s, len(c), f[s], x[s], f"{time.time() - t1:.0f}s", flush=True)
    out = os.path.join(os.environ.get("CURVES_OUT", os.path.join(ROOT, "tests", "golden")), f"curves_mini_{kind}_{seed}.npz")
    np.savez_compressed(out, force=f.astype(np.float32), pos=x, n_plate=nc, digest=dg, n_particles=b.n,
                        settle_s=t1 - t0, run_s=time.time() - t1)
    print("wrote", out, b.n, "particles", f"settle {t1 - t0:.0f}s run {time.time() - t1:.0f}s", flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    kinds = [args[0]] if len(args) > 0 else list(CM.KINDS)
    seeds = [int(args[1])] if len(args) > 1 else list(CM.SEEDS)
    O.set_threads(int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))
    for k in kinds:
        for sd in seeds:
            if "--settled-only" in sys.argv:
                save_settled(k, sd)
            else:
                run(k, sd)
