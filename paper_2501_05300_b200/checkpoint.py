"""Checkpoint and resume of a bed (SURVEY §8(d) bench-bed preparation: "Checkpoint, keyed by
(cfg, variant, seed, code hash)"): particle state in gid order, the contact history (keys and
impulses: the warm start of the next step), and the solver / material / box settings, in one
.npz.  Resuming re-creates the bed through the C-ABI and hands the history back
(dem_set_state), so the continued trajectory is bit-identical to the uninterrupted one.
Plates and moving walls are not part of the checkpoint (their drives are re-issued by the
caller)."""
from __future__ import annotations

import json

import numpy as np

from . import dem as D


def save(bed: "D.Bed", path: str, meta: dict | None = None) -> None:
    if getattr(bed, "_world", 1) > 1:
        raise ValueError("checkpoint a single context (gather the slabs first)")
    st = bed.get_state()
    c = bed.get_contacts()
    cfg = dict(solver={k: (list(v) if isinstance(v, (tuple, list)) else v) for k, v in bed.solver.items()},
               material=dict(bed.material), box={k: (list(v) if isinstance(v, (tuple, list)) else v)
                                                  for k, v in bed.box.items()},
               time=(bed.last_report or {}).get("time", 0.0), meta=meta or {})
    np.savez(path, pos=st["pos"], vel=st["vel"], angvel=st["angvel"], radius=st["radius"], gid=st["gid"],
             hist_key=c["key"], hist_P=c["P"], config=np.frombuffer(json.dumps(cfg).encode(), dtype=np.uint8))


def load(path: str, device: int = 0) -> "D.Bed":
    f = np.load(path)
    cfg = json.loads(bytes(f["config"]).decode())
    sol = dict(cfg["solver"])
    sol["gravity"] = tuple(sol["gravity"])
    box = dict(cfg["box"])
    for k in ("lo", "hi"):
        box[k] = tuple(box[k])
    b = D.Bed(f["pos"], f["radius"], f["vel"], f["angvel"], f["gid"], solver=sol, material=cfg["material"], box=box,
              device=device)
    hist = np.zeros(len(f["hist_key"]), dtype=D.CONTACT_DTYPE)
    hist["key"], hist["P"] = f["hist_key"], f["hist_P"]
    b.set_state(f["pos"], f["radius"], f["vel"], f["angvel"], f["gid"], hist=hist)
    b.checkpoint_meta = cfg.get("meta", {})
    return b
