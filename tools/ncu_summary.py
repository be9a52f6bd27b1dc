"""Summarise an ncu --csv launch list: per-kernel count, total and mean time."""
import csv
import sys
from collections import defaultdict


def summary(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(t for _, t in agg.values())
    out = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  n={n:3d}  mean {t / n / 1e6:8.3f} ms  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
