"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (dev tool)."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows:
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] == "ns" else (v * 1000 if r[ui] == "ms" else v)
        agg[r[ki][:100]].append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{f}: total {tot:.1f} us over {sum(len(v) for v in agg.values())} launches")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:20]:
        print(f"{100 * sum(v) / tot:5.1f}% n={len(v):4d} avg={sum(v) / len(v):8.1f}us  {k}")
