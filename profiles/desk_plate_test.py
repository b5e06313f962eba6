"""Desk-scale paper experiment (SPEC desk preset S:500; PAPER §3.1, §3.3): build a uniform 8.5 mm
bed of the paper's material in a 750 x 120 x 400 mm box with the bed builder (NEXT-2), then run
the plate protocol (NEXT-3) with a 150 mm two-grouser plate (grousers 21.5 mm deep, 12.75 mm
long: the paper's plate halved) under 50 kPa (900 N), phases compressed as the SPEC preset does
(t_I_end 1.5 s, t_II_end 1.75 s, t_end 3.5 s, pull 0.1 m/s ramped over 0.1 s).  Writes the
metrics and a decimated series to gpurun_out/desk_plate_test.json.

The paper's full-scale reference values (1.26 mm static, 70.8 mm dynamic sinkage, traction 0.268
peak / 0.320 average; §4.1-4.2) are for a 300 mm plate on a 1500 x 170 x 600 mm bed: context, not
a target at this scale.

usage: python profiles/desk_plate_test.py [--quick]   (--quick: a 4x smaller box, shorter phases)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_05300_b200 import bedbuilder as BB  # noqa: E402
from paper_2501_05300_b200 import dem as D  # noqa: E402
from paper_2501_05300_b200 import protocol as PR  # noqa: E402


def main():
    quick = "--quick" in sys.argv
    d = 8.5e-3
    dims = (0.375, 0.12, 0.2) if quick else (0.75, 0.12, 0.4)
    t0 = time.perf_counter()
    bed = BB.build_bed(BB.BedSpec(dims=dims, d_min=d, seed=11))
    t_build = time.perf_counter() - t0
    x, r = bed["pos"], bed["radius"]
    n = len(r)
    # plate: base 150 x 118 x 10 mm, two grousers 12.75 mm long, 21.5 mm deep at +-37.5 mm
    L, W, tb, hg, lg = 0.15, 0.118, 0.01, 0.0215, 0.01275
    lo = [(-L / 2, -W / 2, 0.0)] + [(c - lg / 2, -W / 2, -hg) for c in (-0.0375, 0.0375)]
    hi = [(L / 2, W / 2, tb)] + [(c + lg / 2, W / 2, 0.0) for c in (-0.0375, 0.0375)]
    xc = 0.2 if not quick else 0.1
    surf = PR.surface_datum(x, r, (xc, dims[1] / 2), (L / 2, W / 2), cell=2.2 * d)
    z_datum = surf + hg                        # plate height at which the grouser tips touch the surface
    F_N = 50e3 * L * 0.12                      # 50 kPa on the plate footprint (2550 N on 300 x 170 mm)
    proto = PR.PlateProtocol(F_N=F_N, t_ramp=0.5, t_I_end=1.5, u_shear=0.1, t_shear_ramp=0.1, t_II_end=1.75,
                             t_end=3.5) if not quick else \
        PR.PlateProtocol(F_N=F_N / 4, t_ramp=0.2, t_I_end=0.5, u_shear=0.1, t_shear_ramp=0.1, t_II_end=0.65,
                         t_end=1.0, window=0.05)
    rho = BB.PAPER_MATERIAL["density"]
    dt = D.plan_timestep(d, 0.02, rho, 50e3)
    n_it = D.plan_iterations(dims[2] / d, 0.02)
    b = D.Bed(x, r, bed["vel"], bed["angvel"], bed["gid"], solver=dict(dt=dt, n_iter=n_it),
              box=dict(lo=(0, 0, 0), hi=dims, wall_mask=0x3F), material=dict(BB.PAPER_MATERIAL))
    if bed["hist"] is not None:
        b.set_state(x, r, bed["vel"], bed["angvel"], bed["gid"], hist=bed["hist"])
    pid = b.add_plate(lo, hi, (xc, dims[1] / 2, z_datum + 1e-4), 5.0, mu_t=0.3, mu_r=0.02)
    t0 = time.perf_counter()
    series = PR.run_plate_test(b, pid, proto, dt, z_datum)
    t_run = time.perf_counter() - t0
    tm = b.timing() if hasattr(b, "timing") else {}
    b.close()
    m = PR.extract_metrics(series, proto)
    k = max(1, len(series["t"]) // 2000)
    out = dict(particles=n, dims=dims, d=d, dt=dt, n_it=n_it, F_N=F_N, bed_build_wall_s=t_build,
               protocol_wall_s=t_run, steps=len(series["t"]), metrics=m,
               paper_full_scale_reference=dict(static_sinkage=1.26e-3, dynamic_sinkage=70.8e-3, peak_traction=0.268,
                                               avg_traction=0.320),
               series={kk: v[::k].tolist() for kk, v in series.items()})
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "desk_plate_test.json"), "w") as f:
        json.dump(out, f)
    print(json.dumps({kk: v for kk, v in out.items() if kk != "series"}))


if __name__ == "__main__":
    main()
