"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.
usage: python profiles/launch_summary.py gpurun_out/launches.csv profiles/r01_launches.txt "note" """
import csv
import collections
import sys


def main():
    src, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    rows = [r for r in csv.reader(open(src)) if r and not r[0].startswith("==")]
    h = rows[0]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    t = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows[1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0]
        t[name] += float(r[iv].replace(",", ""))
        n[name] += 1
    tot = sum(t.values())
    lines = [f"# ncu launch list summary ({src}); {note}",
             f"# every launch, serialized and cold-cache: compare SHARES, not absolute times",
             f"{'kernel':28s} {'launches':>9s} {'total_ms':>10s} {'mean_us':>9s} {'share':>7s}"]
    for k in sorted(t, key=lambda x: -t[x]):
        lines.append(f"{k:28s} {n[k]:9d} {t[k] / 1e6:10.2f} {t[k] / n[k] / 1e3:9.1f} {100 * t[k] / tot:6.2f}%")
    lines.append(f"{'TOTAL':28s} {sum(n.values()):9d} {tot / 1e6:10.2f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
