"""Summarise an ncu CSV launch list of the 3-D solve kernels: per kernel name and per
launch (time, DRAM bytes)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
launch = collections.OrderedDict()
for d in data:
    key = (d["ID"], d["Kernel Name"])
    launch.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) if d["Metric Value"] else 0.0
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(launch)
items = list(launch.items())[-n:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot_t = tot_b = 0
for (i, name), m in items:
    t = m.get("gpu__time_duration.sum", 0)
    b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    short = name.split("(")[0].split("::")[-1]
    agg[short][0] += 1; agg[short][1] += t; agg[short][2] += b
    tot_t += t; tot_b += b
for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:20s} n={c:4d} time={t/1e3:9.1f} us  dram={b/1e9:7.3f} GB  {b/max(t,1):7.1f} GB/s  share={t/tot_t:.3f}")
print(f"total {tot_t/1e3:.1f} us, {tot_b/1e9:.3f} GB")
