"""Probe: decomposed vs single context when lattice planes drift across a face over many steps
(contacts with impulse history enter a rank's ghost band): max |dv| per setup (diagnostic)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from tests.test_gpu_dist import drifting_bed, single
from tests.parity import run_loopback
for drift, n in ((5.0, 100), (-5.0, 100)):
    bed, box = drifting_bed(drift=drift)
    solver = dict(dt=2e-5, n_iter=30)
    ref = single(bed, n, solver, box)
    out = run_loopback(bed, 2, n, solver, box, bounds=[0.0, 0.0603, 0.12])
    dv = np.abs(out["state"]["vel"] - ref["state"]["vel"]).max()
    print("drift", drift, "steps", n, "max dv", dv, "owned", [r["n_owned"] for r in out["ranks"]])
