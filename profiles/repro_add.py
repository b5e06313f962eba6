import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import synth
from paper_2501_05300_b200 import dem as D
bed = synth.random_cloud(300, (0.005, 0.005, 0.005), (0.035, 0.035, 0.02), 2e-3, 3e-3, 1, v_scale=0.01)
b = D.Bed(bed.x, bed.r, bed.v, bed.w, bed.gid, solver=dict(dt=2e-5, n_iter=20), box=dict(lo=(0, 0, 0), hi=(0.04, 0.04, 0.06)))
gid0 = 1000
try:
    for cyc in range(6):
        b.step(5)
        st = b.get_state(); c = b.get_contacts()
        n_rm = b.remove_particles(2, -np.inf, 0.015)
        print("cycle", cyc, "removed", n_rm, "n", b.n_owned, flush=True)
        ex = synth.random_cloud(40, (0.01, 0.01, 0.03), (0.03, 0.03, 0.05), 0.6e-3 + 0.2e-3 * cyc, 1e-3 + 0.2e-3 * cyc, 2 + cyc)
        b.add_particles(ex.x, ex.r, gid=np.arange(gid0, gid0 + 40)); gid0 += 40
        b.set_solver(n_iter=25 + cyc)
        b.step(5)
        print("cycle", cyc, "ok", b.n_owned, flush=True)
except Exception as e:
    print("ERR", str(e)[:300])
finally:
    b.close()
