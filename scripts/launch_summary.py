"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"].split("(")[0], float(r["Metric Value"]) / 1e3))
    tot = sum(t for _, t in rows)
    agg = collections.OrderedDict()
    for k, t in rows:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    print(f"{len(rows)} launches, {tot:.1f} us total (cold-cache, serialised)")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:<40s} {n:5d} launches {t:10.1f} us  {100 * t / tot:5.1f}%  avg {t / n:9.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
