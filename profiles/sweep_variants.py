"""Time the Jacobi-sweep kernel variants on the bench workload (dem_bench_sweeps diagnostic).

python profiles/sweep_variants.py [--workload config4-geom] [--variants 0,2,10,11,12] [--n 20]
Prints one JSON line per variant: ms per sweep, algorithmic GB/s (SURVEY §8(d) bytes model) and
the max relative velocity difference after n sweeps against the shipped kernel.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config4-geom")
    ap.add_argument("--variants", default="0,2,10,11,12")
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--settle", type=int, default=20)
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    from paper_2501_05300_b200 import dem
    w = bench.WORKLOADS[a.workload]
    b = bench.make_bed(a.workload)
    n_it = dem.plan_iterations(bench.workload_network_length(w), 0.02)
    bed = dem.Bed(b.x, b.r, b.v, b.w, b.gid, device=0, solver=dict(dt=1e-4, n_iter=20),
                  box=dict(lo=b.box_lo, hi=b.box_hi))
    if a.settle:
        bed.step(a.settle)
    bed.set_solver(dt=w["dt"], n_iter=n_it)
    rep = bed.step(1)
    nc = rep["n_contacts"]
    alg = bench.ALG_B_PARTICLE * b.n + bench.ALG_B_CONTACT * nc
    for v in [int(x) for x in a.variants.split(",")]:
        bed.bench_sweeps(v, 3)
        ms, dv = bed.bench_sweeps(v, a.n)
        print(json.dumps({"workload": a.workload, "variant": v, "ms_per_sweep": ms, "alg_GBps": alg / ms / 1e6,
                          "frac_of_peak": alg / ms / 1e6 / bench.peaks().get("hbm_gbs", 6541.1), "max_dv_rel": dv,
                          "n_particles": b.n, "n_contacts": nc}), flush=True)
    bed.close()


if __name__ == "__main__":
    main()
