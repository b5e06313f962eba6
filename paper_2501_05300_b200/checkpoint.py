"""Checkpoint and resume of a bed (SURVEY §8(d) bench-bed preparation: "Checkpoint, keyed by
(cfg, variant, seed, code hash)"): particle state in gid order, the contact history (keys and
impulses: the warm start of the next step), and the solver / material / box settings, in one
.npz.  Resuming re-creates the bed through the C-ABI and hands the history back
(dem_set_state), so the continued trajectory is bit-identical to the uninterrupted one.
Plates, moved walls and the boundary clock are not part of the checkpoint: save() refuses a bed
with a plate or with a wall that has moved or is moving (it would resume with the walls snapped
back to the creation box).  Before the first step the history is empty."""
from __future__ import annotations

import json

import numpy as np

from . import dem as D


def save(bed: "D.Bed", path: str, meta: dict | None = None) -> None:
    if getattr(bed, "_world", 1) > 1:
        raise ValueError("checkpoint a single context (gather the slabs first)")
    if getattr(bed, "n_plates", 0):
        raise ValueError("checkpoint: plates are not captured (save before adding them)")
    lo, hi = bed.box["lo"], bed.box["hi"]
    for wall in range(6):
        if not (bed.box.get("wall_mask", 0x3F) >> wall) & 1:
            continue
        ws = bed.get_wall(wall)
        ax = wall // 2
        home = lo[ax] if wall % 2 == 0 else hi[ax]
        if ws["velocity"] != 0.0 or ws["point"][ax] != home:
            raise ValueError(f"checkpoint: wall {wall} has moved or is moving (walls are not captured)")
    st = bed.get_state()
    try:
        c = bed.get_contacts()
    except D.DemError as e:
        if e.status != D.DEM_ERR_STATE:
            raise
        c = np.zeros(0, dtype=D.CONTACT_DTYPE)          # no step yet: no history
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
