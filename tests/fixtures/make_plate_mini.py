"""Write tests/golden/plate_mini_state.npz: a two-layer refined mini bed (SURVEY §8(d) "c1-mini"
shape: fine 1 mm spheres over the top 0.01 m, 2 mm below; +-10 % radii) in a
0.04 x 0.04 x 0.04 m walled box, settled under gravity in the fp64 ORACLE (h = 1e-4, 20 Jacobi
sweeps).  An INPUT fixture for the plate-curve parity runs, produced only by oracle/ code."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import synth  # noqa: E402


def main(steps=1500, seed=1101):
    b = synth.banded_bed((0.04, 0.04, 0.04), [(0.0, 0.01, 1.0e-3), (0.01, 0.04, 2.0e-3)], seed, spacing=2.25,
                         name="plate-mini")
    W = O.OracleWorld(b.x, b.v, b.w, b.r, b.gid, walls=O.box_walls(b.box_lo, b.box_hi))
    p = O.make_params(h=1e-4, n_it=20)
    t0 = time.time()
    for s in range(steps):
        c, _, _ = W.step(p)
        if s % 250 == 0:
            print(s, b.n, len(c), W.last_report.ke, f"{time.time() - t0:.1f}s", flush=True)
    out = os.path.join(ROOT, "tests", "golden", "plate_mini_state.npz")
    np.savez_compressed(out, x=W.x, v=W.v, w=W.w, r=W.r, gid=W.gid, box_lo=b.box_lo, box_hi=b.box_hi,
                        hist_key=W.hist["key"], hist_P=W.hist["P"], settle_steps=steps, settle_h=1e-4, settle_nit=20,
                        seed=seed)
    print("wrote", out, b.n, "particles", len(W.hist), "contacts; KE", W.last_report.ke)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
