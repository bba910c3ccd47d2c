"""Per-kernel duration summary of an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import OrderedDict


def summarize(path, last=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    seq = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]
    if last:
        seq = seq[-last:]
    agg = OrderedDict()
    for k, v in seq:
        name = k.split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(v)
    tot = sum(v for _, v in seq)
    for k, v in agg.items():
        print(f"{len(v):4d} x {sum(v) / len(v) / 1e3:9.1f} us = {sum(v) / 1e3:9.1f} us ({sum(v) / tot * 100:5.1f}%)  {k}")
    print(f"total {tot / 1e3:.1f} us")
    return seq


if __name__ == "__main__":
    seq = summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else None)
    if "--seq" in sys.argv:
        for k, v in seq:
            print(f"{v / 1e3:9.1f} us  {k.split('(')[0]}")
