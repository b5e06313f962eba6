"""Summarise every kernel launch of an ncu --set full report as one table row (committed evidence
for the kernels besides the sweep): time, DRAM bytes, DRAM throughput, issue activity, occupancy.

usage: python profiles/summarize_many.py gpurun_out/prof_misc.ncu-rep profiles/r01_misc_kernels.txt "note"
"""
import csv
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%pk"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"), ("launch__grid_size", "grid"),
        ("launch__registers_per_thread", "regs")]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    lines = [f"# ncu --set full summary: {rep}", f"# {note}",
             "# units: " + ", ".join(f"{n} [{u[h.index(k)]}]" for k, n in COLS if k in h)]
    lines.append(f"{'kernel':34s} " + " ".join(f"{n:>10s}" for _, n in COLS))
    for v in rows[2:]:
        name = v[h.index("Kernel Name")].split("(")[0][:34]
        cells = [v[h.index(k)] if k in h else "-" for k, _ in COLS]
        lines.append(f"{name:34s} " + " ".join(f"{c:>10s}" for c in cells))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
