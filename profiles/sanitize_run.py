"""Small end-to-end run for compute-sanitizer: walls, a plate, impacts, rebuilds, getters (~60 steps)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2501_05300_b200 import dem  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1500    # 1501: a ragged last tile of odd size
bed = synth.random_cloud(N, (0.002, 0.002, 0.002), (0.058, 0.058, 0.03), 1.0e-3, 3.0e-3, 5, v_scale=0.05, w_scale=3.0,
                         loguniform=True)
b = dem.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=dict(dt=2e-5, n_iter=20),
            box=dict(lo=(0, 0, 0), hi=(0.06, 0.06, 0.06)))
pid = b.add_plate([(-0.01, -0.01, 0.0)], [(0.01, 0.01, 0.003)], (0.03, 0.03, 0.035), 0.05)
b.drive_plate(pid, 2, 1, -0.2)
for _ in range(60):
    rep = b.step(1)
st = b.get_state()
c = b.get_contacts()
F, T = b.get_forces()
print("ok", rep["n_contacts"], rep["impact_fired"], len(c), np.isfinite(F).all(), b.get_plate(pid)["force"])
b.close()
