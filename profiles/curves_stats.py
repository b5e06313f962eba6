"""Statistics of the mini-bed plate curves: per-seed and seed-averaged GPU-vs-oracle
RMS errors, the separation step, and the oracle's own seed-to-seed spread.
    python profiles/curves_stats.py c2 1001 2001 3001 [--gpu-dir gpurun_out]
Reads tests/golden/curves_mini_<kind>_<seed>.npz (oracle) and <gpu-dir>/curves_mini_gpu_<kind>_<seed>.npz."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests import curves_mini as CM  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind")
    ap.add_argument("seeds", nargs="+", type=int)
    ap.add_argument("--gpu-dir", default=os.path.join(ROOT, "gpurun_out"))
    a = ap.parse_args()
    fr = np.array([np.load(os.path.join(ROOT, "tests", "golden", f"curves_mini_{a.kind}_{s}.npz"))["force"].astype(float)
                   for s in a.seeds])
    fg = np.array([np.load(os.path.join(a.gpu_dir, f"curves_mini_gpu_{a.kind}_{s}.npz"))["force"] for s in a.seeds])
    for s, g, r in zip(a.seeds, fg, fr):
        d = np.abs(g - r) / np.abs(r).max()
        print(f"seed {s}: rms {CM.rms_error(g, r):.4f}  max|F| {np.abs(r).max():.3g}  > 1e-6 from step {int(np.argmax(d > 1e-6))}")
    sm = np.array([CM.smooth(r) for r in fr])
    sigma = float(np.sqrt(np.mean(sm.std(axis=0, ddof=1) ** 2)) / np.abs(sm.mean(axis=0)).max())
    n = len(a.seeds)
    print(f"seed-averaged ({n} seeds): rms {CM.rms_error(fg.mean(axis=0), fr.mean(axis=0)):.4f}")
    print(f"oracle seed-to-seed spread {sigma:.4f}; RMS difference of two independent {n}-seed means "
          f"{np.sqrt(2.0 / n) * sigma:.4f}")
    pairs = [CM.rms_error(fr[i], fr[j]) for i in range(n) for j in range(i + 1, n)]
    print("oracle seed-vs-seed rms: min %.4f max %.4f" % (min(pairs), max(pairs)))


if __name__ == "__main__":
    main()
