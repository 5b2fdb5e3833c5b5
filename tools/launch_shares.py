"""Per-kernel launch counts, total time and share from an ncu
`--metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        name = r[ki].split("(")[0].replace("<unnamed>::", "")
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[r[ui]]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v for _, v in agg.values())
    print(f"{'kernel':32s} {'launches':>8s} {'avg us':>10s} {'share':>7s}")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:32s} {n:8d} {v / n:10.1f} {v / tot:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
