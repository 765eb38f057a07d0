"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import sys

SCALE_T = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
SCALE_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                                 "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in data:
        per.setdefault((r[ii], r[ki]), {})[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    out = []
    for (i, k), m in per.items():
        name = k.split("(")[0].replace("hddm::", "").replace("void ", "")
        t, u = m["gpu__time_duration.sum"]
        rb = m.get("dram__bytes_read.sum", (0, "byte"))
        wb = m.get("dram__bytes_write.sum", (0, "byte"))
        out.append((name, t * SCALE_T[u], rb[0] * SCALE_B.get(rb[1], 1), wb[0] * SCALE_B.get(wb[1], 1)))
    return out


def main(path):
    seq = load(path)
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for n, t, r, w in seq:
        a = tot[n]
        a[0] += 1; a[1] += t; a[2] += r; a[3] += w
    s = sum(v[1] for v in tot.values())
    print(f"{'kernel':28s} {'n':>4s} {'us':>10s} {'share':>6s} {'read MB':>9s} {'write MB':>9s} {'GB/s':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        gbs = (v[2] + v[3]) / (v[1] * 1e-6) / 1e9 if v[1] else 0
        print(f"{k:28s} {v[0]:4d} {v[1]:10.1f} {100 * v[1] / s:5.1f}% {v[2] / 1e6:9.1f} {v[3] / 1e6:9.1f} {gbs:7.0f}")
    print(f"total {s:.1f} us")
    if len(sys.argv) > 2:
        for n, t, r, w in seq:
            print(f"  {n:28s} {t:9.1f} us {r / 1e6:8.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1])
