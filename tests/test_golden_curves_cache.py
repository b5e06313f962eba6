"""The cached oracle-settled beds of the mini-curve protocols (tests/golden/curves_mini_<kind>_<seed>_settled.npz,
written by tests/fixtures/make_curves_mini.py --settled-only from the oracle) are the states the stored
oracle curves started from: their digests agree.  CPU only, no oracle run."""
import os

import numpy as np
import pytest

from tests import curves_mini as CM
from tests.fixtures.make_curves_mini import digest, settled_path

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("kind", CM.KINDS)
@pytest.mark.parametrize("seed", CM.SEEDS)
def test_settled_cache_matches_curve_digest(kind, seed):
    cpath = os.path.join(HERE, "golden", f"curves_mini_{kind}_{seed}.npz")
    spath = settled_path(kind, seed)
    if not (os.path.exists(cpath) and os.path.exists(spath)):
        pytest.skip("curve or settled cache not generated")
    z = np.load(spath)

    class W:
        x, v, w = z["x"], z["v"], z["w"]
        hist = z["hist"]

    assert digest(W) == str(z["digest"]) == str(np.load(cpath)["digest"])
    b = CM.make_bed(kind, seed)
    assert len(z["r"]) == b.n and np.array_equal(np.sort(z["gid"]), np.sort(b.gid))
