"""Write tests/golden/config0s_state.npz: config 0 (BASELINE configs[0], synth.config0, seed
1000) settled in the fp64 ORACLE (3,000 steps at h = 1e-4 with 20 Jacobi sweeps).
This is an INPUT fixture (a settled bed for parity runs), produced only by oracle/ code."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import synth  # noqa: E402


def main(steps=3000):
    b = synth.config0(1000)
    W = O.OracleWorld(b.x, b.v, b.w, b.r, b.gid, walls=O.box_walls(b.box_lo, b.box_hi))
    p = O.make_params(h=1e-4, n_it=20)
    for s in range(steps):
        c, _, _ = W.step(p)
        if s % 500 == 0:
            print(s, len(c), W.last_report.ke, flush=True)
    out = os.path.join(ROOT, "tests", "golden", "config0s_state.npz")
    np.savez_compressed(out, x=W.x, v=W.v, w=W.w, r=W.r, gid=W.gid, box_lo=b.box_lo, box_hi=b.box_hi,
                        hist_key=W.hist["key"], hist_P=W.hist["P"], settle_steps=steps, settle_h=1e-4, settle_nit=20)
    print("wrote", out, len(W.hist), "contacts; KE", W.last_report.ke)


if __name__ == "__main__":
    main()
