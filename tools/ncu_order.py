"""Print an ncu --csv launch list in launch order: kernel, grid, us, DRAM MB, GB/s."""
import collections
import csv
import sys


def main(path):
    rows = collections.OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        k = (r["ID"], r["Kernel Name"].split("(")[0], r.get("Grid Size", ""))
        d = rows.setdefault(k, {})
        v = float(r["Metric Value"].replace(",", "") or 0)
        unit = r["Metric Unit"]
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "ms": 1e3, "B": 1e-6, "usecond": 1, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3,
                 "Mbyte": 1, "Gbyte": 1e3}.get(unit, 1)
        d[r["Metric Name"]] = v * scale
    tot = 0
    for (i, name, grid), d in rows.items():
        us = d.get("gpu__time_duration.sum", 0)
        mb = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        tot += us
        print(f"{i:>5} {name[:26]:26s} {grid:>18s} {us:9.1f} {mb:9.1f} {mb / us * 1e-3 if us else 0:8.0f}")
    print("total us", round(tot, 1))


if __name__ == "__main__":
    main(sys.argv[1])
