"""Group an ncu --metrics --csv log by kernel: launches, summed time, DRAM GB, mean L2 hit."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, st = r, i + 1
            break
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = defaultdict(dict)
    for r in rows[st:]:
        if len(r) > vi:
            per[(int(r[ii]), r[ki].split("(")[0])][r[mi]] = float(r[vi].replace(",", ""))
    return per


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        for (i, k), m in sorted(load(p).items()):
            print(f"  {i:3d} {k[:45]:45s} " + "  ".join(f"{n.split('__')[1][:18]}={v:.4g}" for n, v in m.items()))
