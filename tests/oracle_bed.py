"""The fp64 oracle behind the subset of the dem.Bed interface the host-side protocols drive
(test infrastructure: lets tests run bedbuilder / protocol logic on CPU, slowly, on tiny beds)."""
import numpy as np

import oracle as O


class OracleBed:
    def __init__(self, pos, radius, vel=None, angvel=None, gid=None, *, solver=None, box=None, material=None):
        pos = np.asarray(pos, float).reshape(-1, 3)
        n = len(pos)
        vel = np.zeros((n, 3)) if vel is None else vel
        angvel = np.zeros((n, 3)) if angvel is None else angvel
        gid = np.arange(n, dtype=np.uint32) if gid is None else gid
        box = box or {}
        walls = O.box_walls(box.get("lo", (0, 0, 0)), box.get("hi", (1, 1, 1)), mask=box.get("wall_mask", 0x3F),
                            mu_t=box.get("wall_mu_t", 0.0), mu_r=box.get("wall_mu_r", 0.0))
        self.W = O.OracleWorld(pos, vel, angvel, radius, gid, walls=walls)
        m = dict(rho=2600.0, E=1e7, nu=0.3, mu_t=0.4, mu_r=0.1, e_rest=0.5)
        conv = {"density": "rho", "youngs": "E", "poisson": "nu", "restitution": "e_rest"}
        for k, v in (material or {}).items():
            m[conv.get(k, k)] = v
        solver = solver or {}
        self.params = O.make_params(h=solver.get("dt", 1e-5), n_it=solver.get("n_iter", 30), **m)
        self.order = np.argsort(self.W.gid)

    def set_solver(self, n_iter=None, **_):
        if n_iter is not None:
            self.params.n_it = n_iter

    def set_state(self, pos, radius, vel=None, angvel=None, gid=None, hist=None):
        self.W.hist = hist if hist is not None else np.zeros(0, dtype=O.CONTACT_DTYPE)

    def step(self, n=1):
        self.W.step(self.params, n)
        rep = self.W.last_report
        return {"ke": rep.ke, "max_v": rep.max_v, "n_contacts": rep.n_contacts, "time": self.W.time}

    def get_state(self):
        o = self.order
        return {"pos": self.W.x[o].copy(), "vel": self.W.v[o].copy(), "angvel": self.W.w[o].copy(),
                "radius": self.W.r[o].copy(), "gid": self.W.gid[o].copy()}

    def get_contacts(self):
        return self.W.hist.copy()

    def close(self):
        pass
