"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel count / total / share, and optionally the first N launches."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    return [(r[ki].split("(")[0].replace("void ", "").strip(), r[gi], float(r[vi].replace(",", "")))
            for r in rows[hi + 1:] if len(r) > vi]


def main():
    seq = load(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, _, v in seq:
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:44]:44s} {c:8d} {t / 1e3:10.1f} {t / c / 1e3:8.2f} {100 * t / tot:5.1f}%")
    print(f"{'TOTAL':44s} {len(seq):8d} {tot / 1e3:10.1f}")
    for name, g, v in seq[:n]:
        print(f"  {name[:40]:40s} {g:>14s} {v / 1e3:8.1f}")


if __name__ == "__main__":
    main()
