"""c2-mini plate behaviour on the GPU under staggered (0) and monolithic (1) plate coupling:
plate contact count, vertical position and the shear-force curve by windows of 2500 steps.
Settles the bed with the oracle (as tests/test_gpu_z_curves_mini.py does)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from tests import curves_mini as CM  # noqa: E402
from tests.fixtures.make_curves_mini import settled  # noqa: E402
from paper_2501_05300_b200 import dem  # noqa: E402

O.set_threads(os.cpu_count() or 1)
b, W = settled("c2", 1001)
for coupling in (0, 1):
    box = dict(lo=b.box_lo, hi=b.box_hi, wall_mask=CM.WALL_MASK)
    g = dem.Bed(W.x, W.r, W.v, W.w, W.gid, solver=dict(dt=CM.DT, n_iter=CM.N_IT, plate_coupling=coupling), box=box)
    g.set_state(W.x, W.r, W.v, W.w, W.gid, hist=W.hist)
    lo, hi, pos, mass, drives = CM.plate("c2", W.x, W.r, b.box_hi)
    pid = g.add_plate(lo, hi, pos, mass)
    for ax, mode, target, ramp in drives:
        g.drive_plate(pid, ax, mode, target, ramp)
    n = CM.N_STEPS["c2"]
    f = np.empty(n); z = np.empty(n); nc = np.empty(n)
    for s in range(n):
        g.step(1)
        st = g.get_plate(pid)
        f[s], z[s], nc[s] = st["force"][0], st["pos"][2], st.get("n_contacts", 0)
    print("coupling", coupling, "mass", mass, flush=True)
    for i in range(0, n, 2500):
        sl = slice(i, i + 2500)
        print(f"  {i:6d} n_plate {nc[sl].mean():7.1f} z {z[sl].mean():.5f} Fx mean {f[sl].mean():7.2f} std {f[sl].std():6.2f}",
              flush=True)
    g.close()
