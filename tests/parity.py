"""GPU-vs-oracle parity helpers (test infrastructure; used by tests/ and __graft_entry__.smoke).

Both sides receive the same seeded input (synth.Bed) and run the same step independently:
the oracle (fp64 C, brute force) and the CUDA path through the C-ABI binding.  Nothing flows
from the CUDA path into the oracle.

Force/torque error (reading R34): per particle
    err_F = |F_gpu - F_ref| / max(|F_ref|, sum_c |f_c|, m g)
    err_T = |T_gpu - T_ref| / max(|T_ref|, sum_c |tau_c|, r m g)
with f_c, tau_c the oracle's per-contact force and torque on that particle.
"""
from __future__ import annotations

import numpy as np

import oracle as O

G = 9.81


def oracle_world(bed, walls=True, wall_mask=0x3F, plates=(), wall_mu=(0.0, 0.0)):
    W = O.box_walls(bed.box_lo, bed.box_hi, mask=wall_mask, mu_t=wall_mu[0], mu_r=wall_mu[1]) if walls else []
    return O.OracleWorld(bed.x, bed.v, bed.w, bed.r, bed.gid, walls=W, plates=list(plates))


def gpu_bed(bed, walls=True, wall_mask=0x3F, wall_mu=(0.0, 0.0), material=None, **solver):
    from paper_2501_05300_b200 import dem
    box = dict(lo=bed.box_lo, hi=bed.box_hi, wall_mask=wall_mask if walls else 0, wall_mu_t=wall_mu[0],
               wall_mu_r=wall_mu[1])
    return dem.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=solver, box=box, material=material)


def oracle_params(n_it, dt, material=None, **kw):
    m = dict(rho=2600.0, E=1e7, nu=0.3, mu_t=0.4, mu_r=0.1, e_rest=0.5)
    if material:
        conv = {"density": "rho", "youngs": "E", "poisson": "nu", "restitution": "e_rest"}
        for k, v in material.items():
            m[conv.get(k, k)] = v
    return O.make_params(h=dt, n_it=n_it, **m, **kw)


def contact_sums(contacts, bed, h):
    """sum_c |f_c| and sum_c |tau_c| per particle from the oracle's contact list (lever arms
    (r - delta/2) n as in the oracle; reading R10)."""
    n = len(bed.r)
    inv = np.empty(int(bed.gid.max()) + 1 if n else 1, dtype=np.int64)
    inv[bed.gid] = np.arange(n)
    sf = np.zeros(n)
    st = np.zeros(n)
    if len(contacts) == 0:
        return sf, st
    ka = (contacts["key"] >> np.uint64(32)).astype(np.int64)
    kb = (contacts["key"] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    ia = inv[ka]
    Pn, Pt, Pr = contacts["P"][:, 0], contacts["P"][:, 1:4], contacts["P"][:, 4:7]
    nrm, dl = contacts["n"], contacts["delta"]
    L = Pn[:, None] * nrm + Pt
    fa = np.linalg.norm(L, axis=1) / h
    la = (bed.r[ia] - 0.5 * dl)[:, None] * nrm
    ta = np.linalg.norm(np.cross(la, Pt) + Pr, axis=1) / h
    np.add.at(sf, ia, fa)
    np.add.at(st, ia, ta)
    pp = kb < O.PLATE_KEY_BASE
    if pp.any():
        ib = inv[kb[pp]]
        lb = -(bed.r[ib] - 0.5 * dl[pp])[:, None] * nrm[pp]
        tb = np.linalg.norm(np.cross(lb, Pt[pp]) + Pr[pp], axis=1) / h
        np.add.at(sf, ib, fa[pp])
        np.add.at(st, ib, tb)
    return sf, st


def force_errors(F_gpu, T_gpu, F_ref, T_ref, contacts, bed, rho, h):
    """per-particle normalised errors (arrays in gid order)."""
    order = np.argsort(bed.gid)
    r = bed.r[order]
    m = rho * np.pi * (2 * r) ** 3 / 6.0
    sf, st = contact_sums(contacts, bed, h)
    sf, st = sf[order], st[order]
    Fr, Tr = F_ref[order], T_ref[order]
    fl_F = np.maximum.reduce([np.linalg.norm(Fr, axis=1), sf, m * G])
    fl_T = np.maximum.reduce([np.linalg.norm(Tr, axis=1), st, r * m * G])
    eF = np.linalg.norm(F_gpu - Fr, axis=1) / fl_F
    eT = np.linalg.norm(T_gpu - Tr, axis=1) / fl_T
    return eF, eT


def compare_step(bed, n_it=30, dt=1e-5, with_walls=True, hist=None, material=None, n_steps=1, **solver):
    """Run n_steps on both sides from the same state; compare the last step."""
    rho = (material or {}).get("density", 2600.0)
    Wo = oracle_world(bed, walls=with_walls)
    po = oracle_params(n_it, dt, material, **{k: v for k, v in solver.items() if k in ("v_imp", "g", "n_imp", "ordering")})
    gsol = dict(dt=dt, n_iter=n_it)
    if "ordering" in solver:
        gsol["ordering"] = solver["ordering"]
    if "reduction" in solver:
        gsol["reduction"] = solver["reduction"]
    if "v_imp" in solver:
        gsol["v_impact"] = solver["v_imp"]
    if "g" in solver:
        gsol["gravity"] = solver["g"]
    if "n_imp" in solver:
        gsol["n_iter_impact"] = solver["n_imp"]
    gb = gpu_bed(bed, walls=with_walls, material=material, **gsol)
    if hist is not None:
        Wo.hist = hist
        gb.set_state(bed.x, bed.r, bed.v, bed.w, bed.gid, hist=hist)
    try:
        for _ in range(n_steps):
            c_ref, F_ref, T_ref = Wo.step(po, want_forces=True)
            rep = gb.step(1)
        c_gpu = gb.get_contacts()
        F_gpu, T_gpu = gb.get_forces()
        st = gb.get_state()
    finally:
        gb.close()
    pairs_equal = len(c_gpu) == len(c_ref) and np.array_equal(c_gpu["key"], c_ref["key"])
    order = np.argsort(bed.gid)
    eF, eT = force_errors(F_gpu, T_gpu, F_ref, T_ref, c_ref, bed, rho, dt)
    res = {
        "n": len(bed.r), "n_contacts_ref": len(c_ref), "n_contacts_gpu": len(c_gpu), "pairs_equal": bool(pairs_equal),
        "force_err": float(eF.max()) if len(eF) else 0.0, "torque_err": float(eT.max()) if len(eT) else 0.0,
        "force_p99": float(np.percentile(eF, 99)) if len(eF) else 0.0,
        "impact_ref": int(Wo.last_report.impact_fired), "impact_gpu": int(rep["impact_fired"]),
        "n_colors_gpu": int(rep.get("n_colors", 0)),
    }
    if pairs_equal and len(c_ref):
        res["normal_err"] = float(np.abs(c_gpu["n"] - c_ref["n"]).max())
        res["delta_rel_err"] = float((np.abs(c_gpu["delta"] - c_ref["delta"]) / np.maximum(c_ref["delta"], 1e-300)).max())
    vscale = np.abs(Wo.v).max() + 1e-12
    res["v_err_rel"] = float(np.abs(st["vel"] - Wo.v[order]).max() / vscale)
    res["x_err"] = float(np.abs(st["pos"] - Wo.x[order]).max())
    res["detail"] = {"eF": eF, "eT": eT, "c_ref": c_ref, "c_gpu": c_gpu, "state": st, "ref_x": Wo.x[order],
                     "ref_v": Wo.v[order], "ref_w": Wo.w[order]}
    return res


def run_loopback(bed, G, n_steps, solver, box=None, material=None, plates=(), bounds=None, rebalance_every=0):
    """Run bed split into G x-slabs as G loopback ranks of this process (one host thread each,
    include/dem.h dem_loopback_create), n_steps; returns merged state (gid order), the merged
    contact list (key order), per-rank reports and the slab bounds."""
    import threading

    from paper_2501_05300_b200 import dem
    lo, hi = box["lo"], box["hi"]
    if bounds is None:
        bounds = dem.slab_bounds(bed.x[:, 0], G, lo[0], hi[0])
    grp = dem.LoopbackGroup(G)
    res = [None] * G
    err = [None] * G

    def rank_main(r):
        b = None
        try:
            m = (bed.x[:, 0] >= bounds[r]) & (bed.x[:, 0] < bounds[r + 1])
            b = dem.Bed(bed.x[m], bed.r[m], bed.v[m], bed.w[m], bed.gid[m], solver=solver, box=box, material=material,
                        dist=dict(rank=r, world_size=G, slab=(bounds[r], bounds[r + 1]), transport="loopback",
                                  group=grp))
            pids = [b.add_plate(**p) for p in plates]
            reps, faces, owned = [], [], []
            for k in range(n_steps):
                if rebalance_every and k % rebalance_every == 0:
                    faces.append(b.rebalance(256))
                reps.append(b.step(1))
                owned.append(b.n_owned)
            res[r] = dict(state=b.get_state(), contacts=b.get_contacts(), forces=b.get_forces(), reports=reps,
                          faces=faces, owned=owned,
                          plates=[b.get_plate(p) for p in pids], n_local=b.n_local, n_owned=b.n_owned,
                          walls=[b.get_wall(w) for w in range(6) if (box.get("wall_mask", 0x3F) >> w) & 1])
        except Exception as e:   # noqa: BLE001 -- surfaced by the caller
            err[r] = e
        finally:
            if b is not None:
                b.close()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    grp.close()
    for e in err:
        if e is not None:
            raise e
    st = {k: np.concatenate([r["state"][k] for r in res]) for k in res[0]["state"]}
    o = np.argsort(st["gid"])
    st = {k: v[o] for k, v in st.items()}
    F = np.concatenate([r["forces"][0] for r in res])[o]
    T = np.concatenate([r["forces"][1] for r in res])[o]
    c = np.concatenate([r["contacts"] for r in res])
    c = c[np.argsort(c["key"], kind="stable")]
    return dict(state=st, forces=(F, T), contacts=c, ranks=res, bounds=bounds)


def run_loopback_driven(bed, G, n_steps, solver, box, plate, axis, mode, target):
    """run_loopback with one plate whose axis is driven (dem_drive_plate) before the steps."""
    import threading

    from paper_2501_05300_b200 import dem
    bounds = dem.slab_bounds(bed.x[:, 0], G, box["lo"][0], box["hi"][0])
    grp = dem.LoopbackGroup(G)
    res = [None] * G
    err = [None] * G

    def rank_main(r):
        b = None
        try:
            m = (bed.x[:, 0] >= bounds[r]) & (bed.x[:, 0] < bounds[r + 1])
            b = dem.Bed(bed.x[m], bed.r[m], bed.v[m], bed.w[m], bed.gid[m], solver=solver, box=box,
                        dist=dict(rank=r, world_size=G, slab=(bounds[r], bounds[r + 1]), transport="loopback",
                                  group=grp))
            pid = b.add_plate(**plate)
            b.drive_plate(pid, axis, mode, target)
            for _ in range(n_steps):
                b.step(1)
            res[r] = dict(state=b.get_state(), plate=b.get_plate(pid))
        except Exception as e:   # noqa: BLE001 -- surfaced by the caller
            err[r] = e
        finally:
            if b is not None:
                b.close()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    grp.close()
    for e in err:
        if e is not None:
            raise e
    st = {k: np.concatenate([r["state"][k] for r in res]) for k in res[0]["state"]}
    o = np.argsort(st["gid"])
    return dict(state={k: v[o] for k, v in st.items()}, ranks=res)
