"""Oracle side of the mini triaxial: the same servo protocol
(paper_2501_05300_b200/triaxial.py, host logic only) driving the fp64 ORACLE through
tests/oracle_triaxial.py, on the bed and settings of tests/test_gpu_triaxial.py::mini_triaxial.
Writes tests/golden/triaxial_mini_oracle.json (peak deviators and the Mohr-Coulomb fit).
Produced only by oracle/ code:  python tests/fixtures/make_triaxial_oracle.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2501_05300_b200 import triaxial as TX  # noqa: E402
from tests.oracle_triaxial import OracleBed  # noqa: E402
from tests.parity import oracle_params  # noqa: E402

SIGMA3 = (5e3, 15e3, 25e3)


def bed():
    return synth.banded_bed((0.05, 0.05, 0.05), [(0.0, 0.05, 2.5e-3)], 5, spacing=2.1)


def config(s3):
    return TX.TriaxialConfig(sigma3=s3, axial_rate=0.02, max_strain=0.08, K=5e-5, hold=0.01,
                             t_consolidate_max=1.0, smooth=0.01)


def main():
    O.set_binning(True)
    O.set_threads(int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))
    out = {"sigma3": [], "peak": [], "n_particles": 0, "run_s": []}
    for s3 in SIGMA3:
        b = bed()
        ob = OracleBed(b, oracle_params(30, 2e-5, material=dict(mu_t=0.4, mu_r=0.1)), (0, 0, 0), (0.05, 0.05, 0.05))
        t = time.time()
        series = TX.run_triaxial(ob, config(s3), dt=2e-5, record_every=10)
        out["sigma3"].append(s3)
        out["peak"].append(TX.peak_deviator(series, config(s3)))
        out["run_s"].append(time.time() - t)
        out["n_particles"] = len(b.r)
        print(s3, out["peak"][-1], f"{out['run_s'][-1]:.0f}s", flush=True)
    phi, c = TX.mohr_coulomb_fit([(s, s + p) for s, p in zip(out["sigma3"], out["peak"])])
    out["phi_deg"], out["c_pa"] = phi, c
    with open(os.path.join(ROOT, "tests", "golden", "triaxial_mini_oracle.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(out)


if __name__ == "__main__":
    main()
