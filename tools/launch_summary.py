"""Summarise an ncu gpu__time_duration launch list (the --csv --log-file of
`ncu --metrics gpu__time_duration.sum`): per kernel launches and total time
of the LAST run in the file (from the last k_start on).

python tools/launch_summary.py launches.csv [--all]"""
import csv
import sys
from collections import OrderedDict


def load(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    return [(r[ki].split("(")[0].replace("hcc::", ""), float(r[vi].replace(",", "")) / 1e3)
            for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]


def main():
    data = load(sys.argv[1])
    if "--all" not in sys.argv:
        starts = [i for i, (k, _) in enumerate(data) if k == "k_start"]
        if starts:
            data = data[starts[-1]:]
    agg = OrderedDict()
    for k, us in data:
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + us)
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':28s} {'launches':>8s} {'total_us':>10s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:28s} {c:8d} {t:10.1f} {100 * t / tot:6.1f}%")
    print(f"{'sum of kernel time':28s} {len(data):8d} {tot:10.1f}")


if __name__ == "__main__":
    main()
