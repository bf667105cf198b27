"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]).
    python scripts/launch_summary.py gpurun_out/x.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per, names = collections.defaultdict(dict), {}
for r in rows[hi + 1:]:
    per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
    names[r[idi]] = r[ki]


def short(s):
    m = re.search(r"(k_\w+|cub::\w+)", s)
    return m.group(1) if m else s[:40]


agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i in sorted(per, key=int):
    n = short(names[i])
    t = per[i].get("gpu__time_duration.sum", 0) / 1e6
    b = per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0)
    a = agg[n]
    a[0] += 1; a[1] += t; a[2] += b
tot = sum(a[1] for a in agg.values())
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:34s} {c:5d} {t:10.3f} ms {100 * t / tot:5.1f}%  {b / 1e9:8.2f} GB  {b / 1e9 / max(t, 1e-9):6.2f} TB/s")
