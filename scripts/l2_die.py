"""Cluster SMs by L2-hit latency per line (dev tool; reads scripts/micro/l2_die's
lat.bin): prints, per line, the low / high latency split and whether the split is
the same partition of SMs for every line (-> two L2 partitions, SM ids per die)."""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/lat.bin", dtype=np.uint32)
nl, sms = int(raw[0]), int(raw[1])
lat = raw[2:].reshape(256, nl)[:sms].astype(np.float64)
print("latency cycles: min", lat.min(), "median", np.median(lat), "max", lat.max())
# per line: SMs below the line's midpoint between its min and max are "near"
near = np.zeros((sms, nl), dtype=bool)
for i in range(nl):
    col = lat[:, i]
    thr = (col.min() + col.max()) / 2
    near[:, i] = col < thr
# lines whose near-set equals line 0's near-set or its complement
ref = near[:, 0]
same = [(near[:, i] == ref).all() or (near[:, i] == ~ref).all() for i in range(nl)]
print("lines consistent with line 0's partition:", sum(same), "/", nl)
groups = ref
print("SMs near line 0:", int(groups.sum()), np.nonzero(groups)[0].tolist())
print("SMs far from line 0:", int((~groups).sum()), np.nonzero(~groups)[0].tolist())
gap = [lat[~near[:, i], i].mean() - lat[near[:, i], i].mean() for i in range(nl)]
print("mean far - near gap (cycles): %.1f" % float(np.mean(gap)))
