#!/usr/bin/env python
"""bench.py -- throughput of the B200-native nonsmooth-DEM time step (arXiv 2501.05300).

Contract (see the task README): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  A "step" is one full DEM time step (every SURVEY §8(a) row: detection,
history carry, SPOOK rows, impact stage when triggered, N_it Jacobi sweeps, integration with
walls/plates) over the workload bed.  Metric: particle-steps/s (contacts/s reported beside).

Workload (config.workload): BASELINE.json configs[4] "long vehicle-track slab", geom variant
(8.0 x 1.0 x 0.6 m, three refinement bands r = 2 mm to 0.08 m, 6 mm to 0.25 m, 16 mm below,
+-10 % radius jitter), dt = 5e-6 s, N_it from Eqs. 8 + 10 with eps = 0.02.
The bed is a jammed FCC packing (nearest-neighbour distance = mean diameter, so about half
the bonds touch: N_c/N_p ~ 3 like a settled bed), relaxed under gravity for a few coarse
steps (dt 1e-4, 20 sweeps) before the timed steps; see DESIGN.md §4 for the recipe.
Inputs are larger than L2 (several GB per sweep) -> no L2 flush is needed between steps.

N > 1: one process per GPU, x-slab domain decomposition: the bed is
N workload beds laid end to end along x (N x 8 m for config 4), rank r owns the slab
[r L, (r+1) L) and exchanges ghost velocities with its neighbours over NCCL after every Jacobi
sweep (weak scaling: per-GPU work fixed), time = max over ranks.

--impl reference times the fp64 CPU oracle (oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

# SURVEY §8(d); bands = (depth_top, depth_bottom, r_nom)
WORKLOADS = {
    "config4-geom": dict(dims=(8.0, 1.0, 0.6), bands=[(0.0, 0.08, 2e-3), (0.08, 0.25, 6e-3), (0.25, 0.6, 16e-3)],
                         dt=5e-6, seed=1004, plates=8),
    # configs[4]'s stated count (~40 M) on one GPU: the same bands, lengthened along x (reading R27)
    "config4-count": dict(dims=(21.9, 1.0, 0.6), bands=[(0.0, 0.08, 2e-3), (0.08, 0.25, 6e-3), (0.25, 0.6, 16e-3)],
                          dt=5e-6, seed=1004, plates=8),
    "config1": dict(dims=(0.4, 0.4, 0.3), bands=[(0.0, 0.06, 2e-3), (0.06, 0.3, 4e-3)], dt=5e-6, seed=1001),
    "config3-geom": dict(dims=(1.0, 0.5, 0.3), bands=[(0.0, 0.3, 2e-3)], dt=5e-6, seed=1003),
    "config3-count": dict(dims=(4.3, 0.5, 0.3), bands=[(0.0, 0.3, 2e-3)], dt=5e-6, seed=1003),
    # config 2: diameter linear in depth (Eq. 1), d 4 -> 32 mm over the 0.5 m depth (gamma 0.056)
    "config2-geom": dict(dims=(1.0, 0.5, 0.5), profile=(4e-3, 0.056, 32e-3), dt=5e-6, seed=1002),
    "config2-count": dict(dims=(7.8, 0.5, 0.5), profile=(4e-3, 0.056, 32e-3), dt=5e-6, seed=1002),
}
ALG_B_PARTICLE = 112     # algorithmic bytes per particle per sweep (fp64 v, w read + write, statics)
# per contact per sweep at the precision the acceptance demands (SURVEY §8(d)'s own definition):
# n and delta in fp64 (32 B; fp32 normals fail the torque bar) and the impulses
# P_n, P_t, P_r in fp64, read and written (2 x 56 B; fp32 impulses fail it on the bench-shaped
# bed: 6.8e-5).  SURVEY §8(d) budgeted fp32 values: 72 B (reported beside).
ALG_B_CONTACT = 144
ALG_B_CONTACT_SURVEY = 72


def network_length(bands):
    """Eq. 10 generalised to discrete bands: particles along the depth = sum thickness / d."""
    return sum((b - a) / (2 * r) for a, b, r in bands)


def workload_network_length(w):
    """n_d of a workload: discrete bands, or Eq. 10 for the linear profile d = d_min + gamma z
    (capped at d_max): int_0^H dz / d(z)."""
    if "bands" in w:
        return network_length(w["bands"])
    d_min, gamma, d_max = w["profile"]
    H = w["dims"][2]
    z_cap = (d_max - d_min) / gamma
    if z_cap >= H:
        return math.log((d_min + gamma * H) / d_min) / gamma
    return math.log(d_max / d_min) / gamma + (H - z_cap) / d_max


def make_bed(wl, seed_offset=0, spacing=2.0, dims=None):
    """The workload bed on the host (synth); dims overrides the box (bounded oracle samples)."""
    w = WORKLOADS[wl]
    dims = tuple(dims or w["dims"])
    if "profile" in w:
        d_min, gamma, d_max = w["profile"]
        H = dims[2]
        return synth.graded_bed(dims, d_min / 2, min(d_max, d_min + gamma * H) / 2, min(H, (d_max - d_min) / gamma),
                                w["seed"] + seed_offset, spacing=spacing, name=wl)
    return synth.banded_bed(dims, w["bands"], w["seed"] + seed_offset, spacing=spacing, name=wl)


def workload_levels(w):
    """Size classes of the multi-level grid (factor-2 radius bins): bands, or the profile's span."""
    if "bands" in w:
        return len(w["bands"])
    d_min, gamma, d_max = w["profile"]
    return int(math.ceil(math.log2(min(d_max, d_min + gamma * w["dims"][2]) / d_min) - 1e-9))


def make_slab(wl, rank, world):
    """Rank r's slab of the N-long bed: the workload bed (seed per rank) shifted by r L along x
    (synth.shift_slab: gids unique over the job, box spanning all slabs)."""
    return synth.shift_slab(make_bed(wl, seed_offset=rank), rank, world)


def device_generator(wl):
    """The workload bed as an on-device generator (include/dem.h dem_generator, kind bands): the
    same lattice recipe as synth.banded_bed (tests/test_boundary.py checks the site counts)."""
    w = WORKLOADS[wl]
    if "profile" in w:
        d_min, gamma, d_max = w["profile"]
        return dict(kind="profile", d_min=d_min, gamma=gamma, d_max=d_max, spacing_factor=2.0, pos_jitter=0.01,
                    size_jitter=0.10, seed=w["seed"])
    return dict(kind="bands", bands=[(b, r) for (_, b, r) in w["bands"]], spacing_factor=2.0, pos_jitter=0.01,
                size_jitter=0.10, seed=w["seed"])


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, idx):
        self.idx, self.proc, self.path = idx, None, f"/tmp/dem_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        rows = [l.split(",") for l in open(self.path).read().strip().splitlines() if l.strip()]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, n in enumerate(names):
                if r[5 + k].strip() == "Active":
                    reasons.add(n)
        pw = []
        for r in rows:
            try:
                pw.append(float(r[3]))
            except ValueError:
                pass
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][2]), "reasons": sorted(reasons),
                "samples": len(rows), "power_w": float(np.median(pw)) if pw else None}


def cpu_baseline(wl, n_it, dt, budget_s=12.0):
    """The fp64 oracle as it stands (OpenMP over contacts and bodies, bit-identical to its serial
    sweep) on a bounded sample of the workload: a full-depth column of the bed (all bands), stepped
    with the workload's N_it, on all host cores and on one core."""
    import oracle as O
    w = WORKLOADS[wl]
    dims = w["dims"]
    col = (0.06, 0.06, dims[2])
    b = make_bed(wl, seed_offset=77, dims=col)
    O.set_binning(True)                 # the oracle's cell-list mode for timing
    nproc = os.cpu_count() or 1
    legs = {}
    n0 = O.set_threads(0)
    try:
        for cores in (nproc, 1):
            O.set_threads(cores)
            Wd = O.OracleWorld(b.x, b.v, b.w, b.r, b.gid, walls=O.box_walls(b.box_lo, b.box_hi))
            p = O.make_params(h=dt, n_it=n_it)
            t0 = time.perf_counter()
            steps = 0
            while True:
                c, _, _ = Wd.step(p)
                steps += 1
                if time.perf_counter() - t0 > budget_s / 2 or steps >= 3:
                    break
            legs[cores] = (b.n * steps / (time.perf_counter() - t0), steps, len(c))
    finally:
        O.set_threads(n0)
    v, steps, nc = legs[nproc]
    return {"value": v, "unit": "particle-steps/s", "cores": nproc, "nproc": nproc, "kind": "oracle",
            "value_1core": legs[1][0],
            "sample": f"{b.n}-particle full-depth column (0.06 x 0.06 x {dims[2]} m, all bands) of {wl}, "
                      f"{steps} step(s), N_it={n_it}, cell-list (binning) detection, {nc} contacts; OpenMP on "
                      f"{nproc} cores (value) and 1 core (value_1core)"}


def run_reference(args, rank, world):
    wl = args.workload
    w = WORKLOADS[wl]
    n_it = args.n_it or int(np.ceil(0.1 * workload_network_length(w) / 0.02 - 1e-9))
    if rank != 0:
        return
    import oracle as O
    dims = w["dims"]
    b = make_bed(wl, seed_offset=99, dims=(0.05, 0.05, dims[2]))
    O.set_binning(True)                 # the oracle's cell-list mode for timing
    nproc = os.cpu_count() or 1
    O.set_threads(nproc)                # the oracle's OpenMP sweeps on every host core
    Wd = O.OracleWorld(b.x, b.v, b.w, b.r, b.gid, walls=O.box_walls(b.box_lo, b.box_hi))
    p = O.make_params(h=w["dt"], n_it=n_it)
    for _ in range(args.warmup):
        Wd.step(p)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        Wd.step(p)
    T = time.perf_counter() - t0
    val = b.n * args.steps / T
    sample = (f"{b.n}-particle full-depth column (0.05 x 0.05 x {dims[2]} m) of {wl}; each step is one full "
              f"oracle step (cell-list detection, N_it={n_it} Jacobi sweeps), OpenMP on {nproc} cores")
    print(json.dumps({
        "impl": "reference", "metric": "particle-steps/s", "value": val, "unit": "particle-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl + " (oracle sample)", "n_particles": b.n, "n_it": n_it, "dt": w["dt"]},
        "cpu_baseline": {"value": val, "unit": "particle-steps/s", "cores": nproc, "nproc": nproc, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": val, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def torchrun_argv(gpus, argv, port):
    """argv that re-executes this bench under torchrun with one rank per GPU (the contract's own
    launch line), or None when no relaunch is needed (gpus == 1 or already under torchrun)."""
    if gpus <= 1:
        return None
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


# the paper's grouser plate, 0.3 m long (x) across the bed width, 4 teeth 43 mm
# deep x 25.5 mm long at a 75 mm pitch, a 10 mm base; steel density for its mass
def c21_plate_boxes(width):
    hy = 0.5 * width - 0.01
    lo, hi = [(-0.15, -hy, 0.0)], [(0.15, hy, 0.01)]
    for k in range(4):
        xc = -0.1125 + 0.075 * k
        lo.append((xc - 0.01275, -hy, -0.043))
        hi.append((xc + 0.01275, hy, 0.0))
    vol = sum((b[0] - a[0]) * (b[1] - a[1]) * (b[2] - a[2]) for a, b in zip(lo, hi))
    return lo, hi, 7850.0 * vol


def add_plates(bed, n_plates, L_total, width, z_top):
    """n_plates C21 plates evenly along the whole bed, grouser tips 0.1 mm above the bed top
    (every rank adds all of them: plates are global bodies)."""
    lo, hi, mass = c21_plate_boxes(width)
    return [bed.add_plate(lo, hi, ((i + 0.5) * L_total / n_plates, 0.5 * width, z_top + 0.043 + 1e-4), mass)
            for i in range(n_plates)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--workload", default="config4-geom", choices=sorted(WORKLOADS))
    ap.add_argument("--n-it", type=int, default=0)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: one workload bed per GPU (default); strong: the workload bed split into N slabs")
    ap.add_argument("--settle", type=int, default=20)
    ap.add_argument("--settle-dt", type=float, default=1e-4, help="time step of the coarse relaxation (untimed)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no e2e, no baseline, no clocks")
    ap.add_argument("--ordering", default="jacobi", choices=["jacobi", "gs"],
                    help="contact-solve ordering: Jacobi with mass splitting (default) or coloured Gauss-Seidel")
    ap.add_argument("--decompose", action="store_true",
                    help="run the x-slab decomposition (NCCL transport) even at N = 1 (code-path check)")
    ap.add_argument("--plates", default="c21", choices=["c21", "none"],
                    help="c21 (default for config 4): 8 grouser plates pressed (-z) and sheared (+x) at 0.05 m/s in "
                         "the timed window; none: the bed alone")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ:
        relaunch = torchrun_argv(args.gpus, sys.argv[1:], free_port())
        if relaunch:                      # --gpus N without torchrun: one rank per GPU, as the contract launches
            os.execvp(relaunch[0], relaunch)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2501_05300_b200 import dem

    wl = args.workload
    w = WORKLOADS[wl]
    n_it = args.n_it or dem.plan_iterations(workload_network_length(w), 0.02)
    # the bed is generated on the device (dem_generator): N workload beds end to end along x for
    # N ranks, rank r generating the sites of its slab [r L, (r+1) L) under global gids
    # weak: N workload lengths end to end, one per rank; strong: the workload's own bed cut into N slabs
    L_total = w["dims"][0] * (world if args.scaling == "weak" else 1)
    L = L_total / world
    box = dict(lo=(0.0, 0.0, 0.0), hi=(L_total, w["dims"][1], w["dims"][2]))
    gen = device_generator(wl)
    dcfg = None
    if world > 1 or args.decompose:
        obj = [dem.nccl_unique_id() if rank == 0 else None]
        if dist:
            dist.broadcast_object_list(obj, src=0)
        dcfg = dict(rank=rank, world_size=world, slab=(rank * L, (rank + 1) * L), transport="nccl", nccl_id=obj[0])
    bed = dem.Bed(generator=gen, device=local, solver=dict(dt=args.settle_dt, n_iter=20), box=box, dist=dcfg)
    N_total = dem.generator_count(gen, box)
    if args.settle > 0:
        bed.step(args.settle)             # coarse relaxation of the jammed packing (not timed)
    n_plates = w.get("plates", 0) if args.plates == "c21" else 0
    pids = []
    if n_plates:
        # plates start 0.1 mm above the bed; an untimed press at the coarse step brings
        # the grousers ~1.4 mm into the surface, then the window presses (-z) and shears (+x) at 0.05 m/s
        st = bed.get_state()
        z_top = float(np.max(st["pos"][:, 2] + st["radius"])) if len(st["radius"]) else w["dims"][2]
        if dist:
            import torch.distributed as tdist
            zt = torch.tensor([z_top], dtype=torch.float64, device="cuda")
            tdist.all_reduce(zt, op=tdist.ReduceOp.MAX)
            z_top = float(zt.item())
        del st
        pids = add_plates(bed, n_plates, L_total, w["dims"][1], z_top)
        for p in pids:
            bed.drive_plate(p, 2, 1, -0.5)
        bed.step(30)
        for p in pids:
            bed.drive_plate(p, 2, 1, -0.05)
            bed.drive_plate(p, 0, 1, 0.05)
    bed.set_solver(dt=w["dt"], n_iter=n_it, ordering=1 if args.ordering == "gs" else 0)
    wrep = None
    for _ in range(args.warmup):
        wrep = bed.step(1)
    stream = bed.stream
    # timing rule: inputs larger than L2, else flush L2 between timed steps (outside the events)
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    ws = ALG_B_PARTICLE * (N_total / world) + ALG_B_CONTACT * (wrep["n_contacts"] / world if wrep else 0)
    flush = None
    if ws < 2 * l2:
        flush = torch.empty(4 * l2, dtype=torch.uint8, device=f"cuda:{local}")
    l2_note = (f"per-sweep working set {ws / 1e6:.0f} MB < 2 x L2 ({l2 / 1e6:.0f} MB): L2 flushed between timed steps "
               "(4 x L2 written outside the timed events)") if flush is not None else \
        "inputs larger than L2 (no flush needed)"
    bed.set_timing(True)
    bed.reset_timing()
    clocks = ClockSampler(local)
    if not args.profile:
        clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    reps = []
    step_ms = []
    if flush is None:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        evs[0].record(stream)
        for k in range(args.steps):
            reps.append(bed.step(1))
            evs[k + 1].record(stream)
        torch.cuda.synchronize()
        ms = evs[0].elapsed_time(evs[-1])
        step_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    else:
        ev = []
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            reps.append(bed.step(1))
            b.record(stream)
            ev.append((a, b))
        torch.cuda.synchronize()
        step_ms = [a.elapsed_time(b) for a, b in ev]
        ms = sum(step_ms)
    if dist:
        dist.barrier()
    ck = clocks.stop() if not args.profile else None
    tm = bed.timing()
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    N = N_total / world                 # particles per rank (value counts all of them)
    nc_mean = float(np.mean([r["n_contacts"] for r in reps]))
    imp_rate = float(np.mean([r["impact_fired"] for r in reps]))
    rebuild_rate = float(np.mean([r["rebuilt"] for r in reps]))
    value = world * N * args.steps / (ms / 1e3)
    n_imp_sweeps = imp_rate * n_it                 # impact-stage sweeps per step (N_imp = N_it)
    ms_main = ms / args.steps - n_imp_sweeps * (tm["ms_sweeps"] / max(tm["n_sweep_launches"], 1))
    value_main = world * N / (ms_main / 1e3) if ms_main > 0 else None
    # reports are global with the decomposition (each contact counted once over the ranks)
    contacts_per_s = (nc_mean if world > 1 else world * nc_mean) * args.steps / (ms / 1e3)
    nc_rank = nc_mean / world if world > 1 else nc_mean
    sweep_ms = tm["ms_sweeps"] / max(tm["n_sweep_launches"], 1)
    alg_bytes = ALG_B_PARTICLE * N + ALG_B_CONTACT * nc_rank
    pk = peaks()
    hbm = pk.get("hbm_gbs")
    achieved = alg_bytes / (sweep_ms / 1e3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf))[wl]["dram_bytes_per_launch"] / 1e9   # GB per launch (ncu)
        except Exception:
            traffic = None
    out = {
        "metric": "particle-steps/s", "value": value, "unit": "particle-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "ms_per_step_spread": {"min": min(step_ms), "median": float(np.median(step_ms)), "max": max(step_ms),
                               "rank": rank} if step_ms else None,
        "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "n_particles": int(N_total), "generator": "on-device (dem_generator)", "n_contacts_mean": nc_mean, "nc_per_np": nc_mean / N,
                   "n_it": n_it, "dt": w["dt"], "impact_stage_rate": imp_rate, "rebuilds_per_step": rebuild_rate,
                   "levels": workload_levels(w),
                   "device_memory_gb": torch.cuda.max_memory_allocated(local) / 1e9,
                   "parallelism": f"x-slab decomposition x{world} (NCCL ghost exchange per sweep)"
                   if (world > 1 or args.decompose) else "single GPU",
                   "l2": l2_note,
                   "precision": "fp64 state and row math; fp64 normal, overlap and impulse records in the sweep; fp32 contact-array impulses between steps",
                   "ordering": "coloured Gauss-Seidel" if args.ordering == "gs" else "Jacobi (mass splitting)",
                   "reduction": "exact int64 fixed point per particle (order-free: bit-identical for any decomposition)",
                   "plates": n_plates, "plate_contacts_per_step": {"min": min(r["n_plate"] for r in reps),
                                                                   "mean": float(np.mean([r["n_plate"] for r in reps]))},
                   "plate_motion": "kinematic -z 0.05 m/s and +x 0.05 m/s (SURVEY C21: pressed and sheared)"
                   if n_plates else None},
        "value_main_stage_only": value_main,
        "main_stage_only_note": "particle-steps/s with the impact-stage sweeps' time removed, for comparison with "
                                "plate-free settled beds; with the C21 plates moving at 0.05 m/s new plate contacts "
                                "fire the impact stage in nearly every step, and the timed steps include it",
        "contacts_per_s": contacts_per_s,
        "contact_sweeps_per_s": tm["contact_sweeps"] / (ms / 1e3) * world,   # rank-local contacts (incl. ghost copies)
        "roofline": {"bound": "hbm", "kernel": "k_gs_color (all colours of a sweep)" if args.ordering == "gs" else "k_sweep", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": (achieved / hbm) if hbm else None, "traffic": traffic,
                     "traffic_unit": "GB per launch (ncu dram read+write)",
                     "alg_bytes_per_launch": alg_bytes, "launch_ms": sweep_ms,
                     "alg_bytes_model": "112 B/particle + 144 B/contact per sweep: SURVEY 8(d)'s terms at the precision "
                                        "the acceptance demands (fp64 normals and impulses; DESIGN.md 5, 6)",
                     "frac_survey_fp32_model": (ALG_B_PARTICLE * N + ALG_B_CONTACT_SURVEY * nc_rank) / (sweep_ms / 1e3)
                                               / 1e9 / hbm if hbm else None,
                     "sweep_share_of_step": tm["ms_sweeps"] / max(tm["ms_total"], 1e-9),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
                     "frac_vs_8000_GBps": achieved / 8000.0},
        "gpu_launches": int(tm["n_kernel_launches"]),
        "phase_ms_per_step": {k: tm[k] / args.steps for k in ("ms_rebuild", "ms_detect", "ms_sweeps", "ms_integrate")},
    }
    if ck:
        out["clocks"] = ck
    # e2e through the public API (the C-ABI with HOST buffers): per step the drive inputs go H2D
    # (dem_drive_wall / dem_drive_plate upload the boundary state) and dem_get_state copies the
    # whole particle state (a trajectory frame) into pinned host memory
    if not args.no_e2e and not args.profile:
        cap = int(1.2 * N) + 1024        # owned count drifts by migration across the slab faces
        pin = {k: torch.empty((cap, 3), dtype=torch.float64, pin_memory=True) for k in ("pos", "vel", "angvel")}
        n_drive = 4 + 2 * len(pids)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n_own = 0
        for _ in range(args.steps):
            for wall in (0, 1, 2, 3):
                bed.drive_wall(wall, 0.0)            # H2D: boundary drive inputs
            for p in pids:
                bed.drive_plate(p, 2, 1, -0.05)
                bed.drive_plate(p, 0, 1, 0.05)
            bed.step(1)
            n_own = bed.get_state_into(pin)           # D2H through dem_get_state into pinned host buffers
        T = time.perf_counter() - t0
        if dist:
            t = torch.tensor([T], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            T = float(t.item())
        out["e2e"] = {"value": world * N * args.steps / T, "unit": "particle-steps/s",
                      "h2d_bytes_per_step": n_drive * dem.boundary_upload_bytes(), "d2h_bytes_per_step": int(72 * n_own),
                      "what": "per step: wall and plate drive inputs H2D, the full owned particle state (pos, vel, "
                              "angvel; fp64) D2H by dem_get_state into pinned host buffers"}
    if rank == 0 and not args.no_cpu_baseline and not args.profile:
        out["cpu_baseline"] = cpu_baseline(wl, n_it, w["dt"])
    if rank == 0:
        print(json.dumps(out), flush=True)
    bed.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
