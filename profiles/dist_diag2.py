"""Diagnostic: drifting lattice, loopback G ranks vs single context (rows that differ)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from tests.parity import run_loopback  # noqa: E402
from paper_2501_05300_b200 import dem  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
bed = synth.banded_bed((0.12, 0.04, 0.04), [(0.0, 0.04, 2e-3)], 11, spacing=2.05)
bed.v[:, 0] = 5.0
box = dict(lo=(0.0, 0.0, 0.0), hi=(0.12, 0.04, 0.04), wall_mask=0x3C)
solver = dict(dt=2e-5, n_iter=int(os.environ.get("NIT", 30)), v_impact=float(os.environ.get("VIMP", -1)))
for n in ():
    b = dem.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=solver, box=box)
    reps = [b.step(1) for _ in range(n)]
    rs = b.get_state()
    b.close()
    out = run_loopback(bed, G, n, solver, box)
    st = out["state"]
    dv = np.abs(st["vel"] - rs["vel"]).max(axis=1)
    bad = np.nonzero(dv > 1e-12)[0]
    face = out['bounds'][1]
    print('   |x-face| mm of bad:', np.round(np.sort(np.abs(rs['pos'][bad, 0] - face))[:12] * 1e3, 2), 'max dv', dv.max())
    print(f"steps {n}: n_bad {len(bad)} rebuilt {[r['rebuilt'] for r in reps]} bounds {np.round(out['bounds'], 4)} "
          f"nown {[r['n_owned'] for r in out['ranks']]} nlocal {[r['n_local'] for r in out['ranks']]}")
    for i in bad[np.argsort(-dv[bad])][:8]:
        print("   gid", st["gid"][i], "x_single", np.round(rs["pos"][i], 5), "v_single", np.round(rs["vel"][i], 4),
              "x_dist", np.round(st["pos"][i], 5), "v_dist", np.round(st["vel"][i], 4), "dv", dv[i], "x-face mm", round((rs["pos"][i][0] - face) * 1e3, 3))

# grid / history trace of 5 steps (DEM_DEBUG)
if os.environ.get("TRACE"):
    print("=== single"); sys.stdout.flush()
    b = dem.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=solver, box=box)
    for _ in range(5):
        b.step(1)
    b.close()
    print("=== dist"); sys.stdout.flush()
    run_loopback(bed, G, 5, solver, box)
