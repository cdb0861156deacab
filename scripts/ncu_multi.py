"""Summarise an ncu --csv launch list that carries several metrics per launch
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum): per
kernel name, launches, mean us, mean MB read / written, GB/s. Dev tool."""
import collections
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
         "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3}


def main(path: str, last: int = 0) -> None:
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    per = collections.OrderedDict()
    for r in rows:
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1)
    items = list(per.values())[-last:] if last else list(per.values())
    agg = collections.OrderedDict()
    for d in items:
        a = agg.setdefault(d["name"].split("(")[0][:70], [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0)
        a[3] += d.get("dram__bytes_write.sum", 0.0)
    for name, (n, t, rd, wr) in agg.items():
        print(f"{n:4d} {t / n:9.1f} us  rd {rd / n / 1e6:8.1f} MB  wr {wr / n / 1e6:8.1f} MB  "
              f"{(rd + wr) / t / 1e3:7.0f} GB/s  {name}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
