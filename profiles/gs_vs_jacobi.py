"""Convergence of the two orderings on the GPU ("compare iterations-to-residual
against Jacobi at the Eq. 8 N_it"): settled config 0s (tests/golden), one step from the same
state and history, max |P_n - P_n(converged)| / max P_n after N sweeps, the reference being 4,000
Gauss-Seidel sweeps; plus the time per sweep of each ordering on the same bed."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests.parity import gpu_bed  # noqa: E402
from tests.test_gpu_parity import config0s  # noqa: E402

bed, hist = config0s()


def run(n_it, ordering):
    gb = gpu_bed(bed, dt=1e-5, n_iter=n_it, v_impact=1e30, ordering=ordering)
    gb.set_state(bed.x, bed.r, bed.v, bed.w, bed.gid, hist=hist)
    gb.set_timing(True)
    gb.reset_timing()
    rep = gb.step(1)
    tm = gb.timing()
    c = gb.get_contacts()
    gb.close()
    return c["P"][:, 0], tm["ms_sweeps"] / max(n_it, 1), rep


ref, _, _ = run(4000, 1)
scale = ref.max()
print(f"config 0s: {len(bed.r)} particles, {len(ref)} contacts; reference = 4000 Gauss-Seidel sweeps")
print(f"{'N_it':>6s} {'Jacobi err':>12s} {'GS err':>12s} {'Jacobi ms/sweep':>16s} {'GS ms/sweep':>12s} colours")
for n in (5, 10, 20, 46, 92, 184, 368):
    pj, tj, _ = run(n, 0)
    pg, tg, rg = run(n, 1)
    print(f"{n:6d} {np.abs(pj - ref).max() / scale:12.3e} {np.abs(pg - ref).max() / scale:12.3e} {tj:16.4f} {tg:12.4f} "
          f"{rg['n_colors']}", flush=True)
