"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def main(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0].split("::")[-1]
        if k.startswith("<unnamed>"):
            k = r[ki].split("(")[0].split(">::")[-1]
        t = float(r[vi].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':28s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:28s} {n:8d} {t / 1e3:10.1f} {t / n / 1e3:9.1f} {100 * t / tot:5.1f}%")
    print(f"{'total':28s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
