"""Small-bed step time with and without CUDA-graph replay of the sweep loops (run twice: with
DEM_NO_GRAPHS=1 and without).  Config 0 (4,096 spheres, 92 sweeps) and config 1 sized beds."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2501_05300_b200 import dem

import numpy as np
import oracle as O
f = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "config0s_state.npz"))
c0s = synth.Bed(x=f["x"], r=f["r"], v=f["v"], w=f["w"], gid=f["gid"], box_lo=tuple(f["box_lo"]), box_hi=tuple(f["box_hi"]))
for name, bed, dt, nit in (("config0s (settled)", c0s, 1e-5, 92),):
    b = dem.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=dict(dt=dt, n_iter=nit), box=dict(lo=bed.box_lo, hi=bed.box_hi))
    b.step(20)
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = b.step(200)
    torch.cuda.synchronize()
    el = (time.perf_counter() - t) / 200
    print(name, "graphs" if not os.environ.get("DEM_NO_GRAPHS") else "no graphs", f"{el * 1e3:.3f} ms/step",
          "impact", rep["impact_fired"], "contacts", rep["n_contacts"])
    b.close()
