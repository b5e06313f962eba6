import sys
sys.path.insert(0, "/root/repo")
from paper_2501_05300_b200 import bedbuilder as BB
orig_run, orig_add, orig_open = BB._World.run_until, BB._World.add, BB._World.open
def run(self, *a, **k):
    print("run_until n", len(self.r), "t", round(self.t, 3), "n_iter", getattr(self, "n_iter_now", None), flush=True)
    return orig_run(self, *a, **k)
BB._World.run_until = run
spec = BB.BedSpec(dims=(0.1, 0.1, 0.06), d_min=0.006, d_max=0.0104, r=1.2, eta=2.0, seed=4)
try:
    out = BB.build_bed(spec)
    print("OK", len(out["radius"]))
except Exception as e:
    print("ERR", e)
