"""Time the rebuild phase (keys, sort, grid, broad phase, history carry) on a bench workload:
DEM_LIB_VARIANT=<libdem.so> python profiles/rebuild_timing.py --tag T.  Steps the unsettled bed as
profiles/sweep_ab.py prepares it (dt 1e-4, 20 sweeps) and prints the dem-timed rebuild phase of
every step that rebuilt, as one JSON line."""
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
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    from paper_2501_05300_b200 import dem
    w = bench.WORKLOADS[a.workload]
    box = dict(lo=(0.0, 0.0, 0.0), hi=tuple(w["dims"]))
    bed = dem.Bed(generator=bench.device_generator(a.workload), device=0, solver=dict(dt=1e-4, n_iter=20), box=box)
    bed.set_timing(True)
    ms = []
    for _ in range(a.n):
        bed.reset_timing()
        rep = bed.step(1)
        if rep["rebuilt"]:
            ms.append(bed.timing()["ms_rebuild"])
    print(json.dumps({"tag": a.tag, "lib": os.environ.get("DEM_LIB_VARIANT", "default"), "workload": a.workload,
                      "ms_rebuild": ms}), flush=True)
    bed.close()


if __name__ == "__main__":
    main()
