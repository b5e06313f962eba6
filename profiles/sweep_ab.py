"""Time the shipped sweep kernel (dem_bench_sweeps) on a bench workload, for A/B comparisons of
build variants: DEM_LIB_VARIANT=<path to libdem.so> python profiles/sweep_ab.py --tag T.
Prints one JSON line (ms per sweep sustained over --n sweeps, after the bench's preparation)."""
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
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--tag", default="")
    ap.add_argument("--settle", type=int, default=20)
    a = ap.parse_args()
    import torch
    from paper_2501_05300_b200 import dem
    w = bench.WORKLOADS[a.workload]
    n_it = dem.plan_iterations(bench.workload_network_length(w), 0.02)
    box = dict(lo=(0.0, 0.0, 0.0), hi=tuple(w["dims"]))
    bed = dem.Bed(generator=bench.device_generator(a.workload), device=0, solver=dict(dt=1e-4, n_iter=20), box=box)
    bed.step(a.settle)
    bed.set_solver(dt=w["dt"], n_iter=n_it)
    rep = bed.step(2)
    bed.bench_sweeps(0, 5)
    ms, _ = bed.bench_sweeps(0, a.n)
    N = dem.generator_count(bench.device_generator(a.workload), box)
    nc = rep["n_contacts"]
    alg = bench.ALG_B_PARTICLE * N + bench.ALG_B_CONTACT * nc
    alg72 = bench.ALG_B_PARTICLE * N + bench.ALG_B_CONTACT_SURVEY * nc
    pk = bench.peaks().get("hbm_gbs")
    print(json.dumps({"tag": a.tag, "lib": os.environ.get("DEM_LIB_VARIANT", "default"), "workload": a.workload,
                      "ms_per_sweep": ms, "n_particles": N, "n_contacts": nc,
                      "achieved_GBps": alg / (ms / 1e3) / 1e9, "frac": alg / (ms / 1e3) / 1e9 / pk if pk else None,
                      "frac_survey72": alg72 / (ms / 1e3) / 1e9 / pk if pk else None}),
          flush=True)
    bed.close()


if __name__ == "__main__":
    main()
