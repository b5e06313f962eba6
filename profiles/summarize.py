"""Summarise an ncu report of the sweep kernel into profiles/<name>.txt (committed evidence).

usage: python profiles/summarize.py gpurun_out/prof.ncu-rep profiles/r01_sweep_vX.txt "note"
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum"]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    lines = [f"# ncu --set full summary: {rep}", f"# {note}", f"kernel: {v[h.index('Kernel Name')]}"]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append(f"{k:62s} {v[i]:>18s} {u[i]}")
    stalls = [(n, v[i]) for i, n in enumerate(h)
              if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
    stalls.sort(key=lambda t: -float(t[1] or 0))
    lines.append("top stall reasons (pc samples):")
    for n, val in stalls[:8]:
        lines.append(f"  {n.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {val}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
