"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv).  The one-time
setup kernels (device-resident numeric setup, dsetup.cu) are listed apart and excluded from the
shares, which are shares of the timed sweeps."""
import collections
import csv
import sys


SETUP = {"factor_kernel", "aux_entries_kernel", "aux_diag_kernel", "sc_cell_data_kernel"}


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"].split("(")[0], float(r["Metric Value"]) / 1e3))
    setup = [(k, t) for k, t in rows if k.split("::")[-1] in SETUP]
    rows = [(k, t) for k, t in rows if k.split("::")[-1] not in SETUP]
    tot = sum(t for _, t in rows)
    agg = collections.OrderedDict()
    for k, t in rows:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    print(f"{len(rows)} launches, {tot:.1f} us total (cold-cache, serialised)")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:<40s} {n:5d} launches {t:10.1f} us  {100 * t / tot:5.1f}%  avg {t / n:9.1f} us")
    if setup:
        print(f"setup (once, not in the shares): " + ", ".join(f"{k.split('::')[-1]} {t / 1e3:.1f} ms" for k, t in setup))


if __name__ == "__main__":
    main(sys.argv[1])
