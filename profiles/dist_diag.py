"""Diagnostic: loopback decomposition vs single context, step by step (prints where they differ)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from tests.parity import run_loopback  # noqa: E402
from paper_2501_05300_b200 import dem  # noqa: E402


def single(bed, n, solver, box):
    b = dem.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=solver, box=box)
    reps = [b.step(1) for _ in range(n)]
    st = b.get_state()
    b.close()
    return st, reps


kind = sys.argv[1] if len(sys.argv) > 1 else "cloud"
if kind == "cloud":
    bed = synth.random_cloud(3000, (0.002, 0.002, 0.002), (0.118, 0.038, 0.058), 1.0e-3, 2.4e-3, 3, v_scale=0.05, w_scale=5.0)
    box = dict(lo=(0.0, 0.0, 0.0), hi=(0.12, 0.04, 0.06))
else:
    bed = synth.banded_bed((0.12, 0.04, 0.04), [(0.0, 0.04, 2e-3)], 11, spacing=2.05)
    box = dict(lo=(0.0, 0.0, 0.0), hi=(0.12, 0.04, 0.04))
solver = dict(dt=2e-5, n_iter=30)
for n in (1, 2, 3, 6):
    rs, reps = single(bed, n, solver, box)
    out = run_loopback(bed, 2, n, solver, box)
    st = out["state"]
    dv = np.abs(st["vel"] - rs["vel"]).max(axis=1)
    bad = np.nonzero(dv > 1e-9 * np.abs(rs["vel"]).max())[0]
    face = out["bounds"][1]
    print(f"steps {n}: max|dv| {dv.max():.3e} vmax {np.abs(rs['vel']).max():.3e} n_bad {len(bad)} "
          f"impact {[r['impact_fired'] for r in reps]} rebuilt {[r['rebuilt'] for r in reps]} "
          f"contacts {reps[-1]['n_contacts']} vs {[r['reports'][-1]['n_contacts'] for r in out['ranks']]} "
          f"nlocal {[r['n_local'] for r in out['ranks']]} nown {[r['n_owned'] for r in out['ranks']]}")
    if len(bad):
        print("   bad |x - face| (mm):", np.round(np.abs(rs["pos"][bad, 0] - face) * 1e3, 2)[:20])
