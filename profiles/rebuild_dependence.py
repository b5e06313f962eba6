"""Probe: is the decomposed trajectory bit-identical to the single context when slab faces move
(dem_rebalance)?  Prints the first step with a difference and the particles involved (diagnostic)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from tests.test_gpu_dist import drifting_bed, single
from tests.parity import run_loopback

bed, box = drifting_bed(drift=0.0, seed=9)
solver = dict(dt=2e-5, n_iter=20)
for n in range(1, 16):
    ref = single(bed, n, solver, box)
    b = run_loopback(bed, 3, n, solver, box, bounds=[0.0, 0.02, 0.04, 0.12], rebalance_every=1)
    db = np.abs(b["state"]["pos"] - ref["state"]["pos"]).max(axis=1)
    dv = np.abs(b["state"]["vel"] - ref["state"]["vel"]).max(axis=1)
    if dv.max() > 0:
        bad = np.flatnonzero(dv > 0)
        print("step", n, "n_bad", len(bad), "faces", b["ranks"][0]["faces"][-2:], "owned", [r["owned"][-2:] for r in b["ranks"]])
        for i in bad[np.argsort(-dv[bad])][:8]:
            print("  gid", ref["state"]["gid"][i], "x", ref["state"]["pos"][i], "dv", dv[i])
        ck = b["contacts"]; cr = ref["contacts"]
        print("  contacts equal keys", np.array_equal(ck["key"], cr["key"]), len(ck), len(cr))
        if np.array_equal(ck["key"], cr["key"]):
            dP = np.abs(ck["P"] - cr["P"]).max(axis=1)
            for j in np.argsort(-dP)[:5]:
                print("  key", int(cr["key"][j]) >> 32, int(cr["key"][j]) & 0xFFFFFFFF, "dP", dP[j], "P", cr["P"][j][:2], ck["P"][j][:2])
        break
    print("step", n, "identical", "faces", b["ranks"][0]["faces"][-1])
