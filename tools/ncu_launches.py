"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch
list: per kernel name, count / total / mean device time and share.
usage: python tools/ncu_launches.py launches.csv [--list]"""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
        out.append((r[ki].split("(")[0], v * scale))
    return out


def main(path, listing=False):
    L = load(path)
    if listing:
        for name, us in L:
            print(f"{us:10.2f} us  {name}")
        return
    tot, cnt = defaultdict(float), defaultdict(int)
    for name, us in L:
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'total us':>10} {'share':>6} {'n':>5} {'mean us':>9}  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.1f} {100 * v / T:5.1f}% {cnt[k]:5d} {v / cnt[k]:9.2f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], "--list" in sys.argv)
