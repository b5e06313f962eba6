"""Force/torque parity errors of the current library (DEM_LIB_VARIANT selects a build) on the
one-step parity cases of tests/test_gpu_parity.py: prints max and p99 of the normalised errors."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from tests.parity import compare_step  # noqa: E402
from tests.test_gpu_parity import config0s  # noqa: E402

cases = []
for seed in (1, 2, 3):
    cases.append((f"cloud{seed}", synth.random_cloud(600, (0, 0, 0), (0.05, 0.05, 0.05), 1.5e-3, 3.5e-3, seed,
                                                     v_scale=0.02, w_scale=2.0), dict(n_it=40, dt=1e-5)))
cases.append(("poly8x", synth.random_cloud(800, (0, 0, 0), (0.08, 0.08, 0.08), 1e-3, 8e-3, 9, v_scale=0.01,
                                           loguniform=True), dict(n_it=40, dt=1e-5)))
cases.append(("config0x3", synth.config0(), dict(n_it=92, dt=1e-5, n_steps=3)))
bed, hist = config0s()
cases.append(("config0s", bed, dict(n_it=92, dt=1e-5, hist=hist, v_imp=1e30)))
worst = {"force": 0.0, "torque": 0.0}
for name, b, kw in cases:
    r = compare_step(b, **kw)
    eF, eT = r["detail"]["eF"], r["detail"]["eT"]
    worst["force"] = max(worst["force"], r["force_err"])
    worst["torque"] = max(worst["torque"], r["torque_err"])
    print(json.dumps({"case": name, "pairs_equal": r["pairs_equal"], "force_max": r["force_err"],
                      "torque_max": r["torque_err"], "force_p99": float(np.percentile(eF, 99)),
                      "torque_p99": float(np.percentile(eT, 99))}), flush=True)
print(json.dumps({"lib": os.environ.get("DEM_LIB_VARIANT", "libdem.so"), "worst": worst}))
