"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV):
per-kernel count, total/avg device time and share, optionally restricted
to the last N launches (the timed decode steps)."""
import csv
import sys
from collections import defaultdict


def main(path, last=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    launches = []
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        try:
            launches.append((r[ki].split("(")[0].replace("(anonymous namespace)::", ""), float(r[vi].replace(",", ""))))
        except ValueError:
            pass
    if last:
        launches = launches[-int(last):]
    agg = defaultdict(lambda: [0, 0.0])
    for n, t in launches:
        agg[n][0] += 1
        agg[n][1] += t
    tot = sum(v[1] for v in agg.values())
    print(f"{len(launches)} launches, total {tot / 1e3:.1f} us (ncu: serialised, cold caches - compare shares)")
    print(f"{'kernel':70s} {'n':>5s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:70]:70s} {n:5d} {t / 1e3:10.1f} {t / n / 1e3:9.2f} {t / tot * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
