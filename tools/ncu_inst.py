"""Per kernel family: time, warp / thread instructions and DFMA count from an ncu
--metrics CSV (long format). Usage: ncu_inst.py launches.csv [n_last]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "ID")
per = collections.OrderedDict()
for r in rows:
    if len(r) != len(hdr) or r[0] == "ID":
        continue
    d = dict(zip(hdr, r))
    k = per.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0]})
    k[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
ks = list(per.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(ks) // 2
ks = ks[-n:]
fam = collections.OrderedDict()
for k in ks:
    f = fam.setdefault(k["name"], collections.Counter())
    f["n"] += 1
    for m in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
              "lts__t_bytes.sum", "dram__bytes_read.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"):
        f[m] += k.get(m, 0)
    f["wa"] += k.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0) * k["gpu__time_duration.sum"]
tot = collections.Counter()
print(f"{'family':16s} {'n':>4s} {'us':>8s} {'Mwinst':>8s} {'lanes/wi':>8s} {'cfma(M)':>8s} {'slots/cfma':>10s} {'thr/cfma':>8s} {'L2 GB':>6s} {'warps%':>6s}")
for name, f in fam.items():
    cf = f["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"] / 4
    wi = f["smsp__inst_executed.sum"]
    ti = f["smsp__thread_inst_executed.sum"]
    print(f"{name:16s} {f['n']:4d} {f['gpu__time_duration.sum']/1e3:8.1f} {wi/1e6:8.1f} {ti/max(wi,1):8.1f} "
          f"{cf/1e6:8.1f} {32*wi/max(cf,1):10.1f} {ti/max(cf,1):8.1f} {f['lts__t_bytes.sum']/1e9:6.2f} "
          f"{f['wa']/max(f['gpu__time_duration.sum'],1):6.1f}")
    tot.update(f)
cf = tot["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"] / 4
print(f"{'total':16s} {tot['n']:4d} {tot['gpu__time_duration.sum']/1e3:8.1f} {tot['smsp__inst_executed.sum']/1e6:8.1f} "
      f"{'':8s} {cf/1e6:8.1f} {32*tot['smsp__inst_executed.sum']/cf:10.1f} {tot['smsp__thread_inst_executed.sum']/cf:8.1f} "
      f"{tot['lts__t_bytes.sum']/1e9:6.2f}")
