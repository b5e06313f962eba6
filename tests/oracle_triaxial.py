"""The fp64 oracle behind the dem.Bed calls the triaxial protocol uses (step, get_wall,
drive_wall), so paper_2501_05300_b200/triaxial.py drives the ORACLE through the same servo
protocol as the GPU.  Test infrastructure: only tests/ import it.

Wall w = 2 axis + side, inward normals; a wall's reaction is the oracle's own contact impulses
summed over its contacts, F_w = sum (P_n n + P_t) / h (the dem_get_wall convention, checked
against the GPU in tests/test_gpu_triaxial.py::test_wall_reaction_sums)."""
import numpy as np

import oracle as O


class OracleBed:
    def __init__(self, bed, params, lo, hi):
        self.W = O.OracleWorld(bed.x, bed.v, bed.w, bed.r, bed.gid, walls=O.box_walls(lo, hi))
        self.p = params
        self.force = np.zeros((6, 3))
        self.count = np.zeros(6, dtype=np.int64)

    def step(self, n=1):
        c, _, _ = self.W.step(self.p, n)
        lo = (c["key"] & np.uint64(0xFFFFFFFF)).astype(np.int64)
        for w in range(6):
            m = lo == O.WALL_KEY_BASE + w
            P = c["P"][m]
            self.force[w] = (P[:, :1] * c["n"][m] + P[:, 1:4]).sum(axis=0) / self.p.h
            self.count[w] = int(m.sum())

    def get_wall(self, w):
        wl = self.W.walls[w]
        return {"point": list(wl.p), "normal": list(wl.n), "force": self.force[w].tolist(), "velocity": wl.vel,
                "n_contacts": int(self.count[w])}

    def drive_wall(self, w, v):
        self.W.walls[w].vel = float(v)

    def close(self):
        pass
