"""bench.py contract on CPU: the reference arm (the fp64 oracle on a bounded sample of the bench
workload) prints one JSON line with the contract's keys; the GPU arm's argument parsing."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "particle-steps/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("config4-geom")


def test_workload_iteration_counts():
    """N_it of every bench workload from Eqs. 8 + 10: bands sum thickness / d; the
    Eq. 1 profile integrates dz / d(z) (numerically here, against the closed form in bench.py);
    config 4 and config 2 reproduce SURVEY §8(d)'s 226 and 186."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    from paper_2501_05300_b200 import dem
    w2 = bench.WORKLOADS["config2-geom"]
    d_min, gamma, d_max = w2["profile"]
    z = np.linspace(0.0, w2["dims"][2], 200001)
    d = np.minimum(d_max, d_min + gamma * z)
    f = 1.0 / d
    num = float(np.sum(0.5 * (f[1:] + f[:-1]) * np.diff(z)))
    assert abs(bench.workload_network_length(w2) - num) < 1e-6 * num
    assert dem.plan_iterations(bench.workload_network_length(bench.WORKLOADS["config4-geom"]), 0.02) == 226
    assert dem.plan_iterations(bench.workload_network_length(w2), 0.02) == 186
    assert dem.plan_iterations(bench.workload_network_length(bench.WORKLOADS["config3-count"]), 0.02) == 375
    assert bench.workload_levels(w2) == 3 and bench.workload_levels(bench.WORKLOADS["config4-geom"]) == 3


def test_gpus_flag_relaunches_one_rank_per_gpu():
    """VERDICT r1 / ADVICE: `bench.py --gpus N` without torchrun re-executes itself under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous); a WORLD_SIZE that disagrees with
    --gpus is refused.  Exercised on CPU through the reference arm (rank 0 alone prints)."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench.torchrun_argv(1, ["--gpus", "1"], 29500) is None
    argv = bench.torchrun_argv(4, ["--gpus", "4", "--steps", "2"], 29511)
    assert argv[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "--master-port=29511" in argv
    assert argv[argv.index("--master-addr") + 1] == "127.0.0.1"
    assert argv[-4:] == ["--gpus", "4", "--steps", "2"] and argv[-5].endswith("bench.py")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2
    env["WORLD_SIZE"] = "2"
    bad = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1"], capture_output=True,
                         text=True, timeout=120, cwd=ROOT, env=env)
    assert bad.returncode != 0 and "WORLD_SIZE=2" in (bad.stderr + bad.stdout)
