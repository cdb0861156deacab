"""Per-CUDA-line warp-stall samples from `ncu --page source --csv --print-source cuda,sass` (dev tool)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = next(i for i, x in enumerate(rows) if "Warp Stall Sampling (All Samples)" in x)
h = rows[hi]
wi = h.index("Warp Stall Sampling (All Samples)")
agg = collections.Counter()
src = {}
line = None
for x in rows[hi + 1:]:
    if len(x) <= wi:
        continue
    if x[0]:
        line = x[0]
        src[line] = x[1][:100]
    try:
        agg[line] += float(x[wi] or 0)
    except ValueError:
        pass
tot = sum(agg.values()) or 1
for l, v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% L{l}: {src.get(l, '')}")
