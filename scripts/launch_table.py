"""Markdown table of a multi-metric ncu launch list (gpu__time_duration + DRAM bytes),
library kernels only (dev tool): python scripts/launch_table.py launches.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
h = rows[hi]
ki, ii, mi, ui, vi = (h.index(c) for c in ("Kernel Name", "ID", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = collections.defaultdict(dict)
name = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    per[r[ii]][r[mi]] = v
    name[r[ii]] = r[ki]


def short(n: str) -> str:
    n = re.sub(r"\(.*", "", n).replace("void ", "")
    return n


agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in per.items():
    n = short(name[i])
    if not (n.startswith("i8mm::") or n.startswith("gemm::")):
        continue
    a = agg[n]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print("| share | launches | avg us | avg DRAM rd MB | avg DRAM wr MB | GB/s | kernel |")
print("|---:|---:|---:|---:|---:|---:|---|")
for n, (c, t, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {100 * t / tot:.1f}% | {c} | {t / c:.1f} | {rd / c / 1e6:.1f} | {wr / c / 1e6:.1f} | "
          f"{(rd + wr) / t / 1e3:.0f} | `{n}` |")
