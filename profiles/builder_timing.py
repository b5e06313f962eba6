"""Wall time of the bed builder (host orchestration + library) on a mid-size uniform bed."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_05300_b200 import bedbuilder as BB
from paper_2501_05300_b200.protocol import surface_datum

dims = tuple(float(v) for v in (sys.argv[1:4] if len(sys.argv) >= 4 else (0.3, 0.12, 0.15)))
d = float(sys.argv[4]) if len(sys.argv) >= 5 else 8.5e-3
t = time.perf_counter()
out = BB.build_bed(BB.BedSpec(dims=dims, d_min=d, seed=1))
el = time.perf_counter() - t
H = surface_datum(out["pos"], out["radius"], (dims[0] / 2, dims[1] / 2), (dims[0] / 2, dims[1] / 2), cell=2.2 * d)
print(f"dims {dims} d {d}: n {len(out['radius'])} surface {H:.4f} t_sim {out['t_sim']:.2f} s dt {out['dt']:.2e} wall {el:.1f} s")
