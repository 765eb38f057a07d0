"""Per-launch unit throughputs from an ncu --csv metrics list (scratch/thr.sh)."""
import collections
import csv
import sys


def main(path, min_us=15.0):
    rows = collections.OrderedDict()
    lines = [l for l in open(path) if l.startswith('"')]
    for r in csv.DictReader(lines):
        k = (r["ID"], r["Kernel Name"].split("(")[0].replace("void ", "").replace("hddm::", ""),
             r.get("Grid Size", ""))
        rows.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "") or 0)
    print(f"{'kernel':22s} {'grid':>14s} {'us':>7s} {'dramMB':>7s} {'L1%':>5s} {'L2%':>5s} {'DR%':>5s} "
          f"{'SM%':>5s} {'sec/rq':>6s} {'occ%':>5s}")
    tot = collections.defaultdict(float)
    for (i, n, g), d in rows.items():
        us = d["gpu__time_duration.sum"] / 1e3
        dr = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / 1e6
        sr = d["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"] / max(
            1, d["l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"])
        tot[n] += us
        if us >= min_us:
            print(f"{n[:22]:22s} {g:>14s} {us:7.1f} {dr:7.1f} "
                  f"{d['l1tex__throughput.avg.pct_of_peak_sustained_elapsed']:5.1f} "
                  f"{d['lts__throughput.avg.pct_of_peak_sustained_elapsed']:5.1f} "
                  f"{d['dram__throughput.avg.pct_of_peak_sustained_elapsed']:5.1f} "
                  f"{d['sm__throughput.avg.pct_of_peak_sustained_elapsed']:5.1f} {sr:6.1f} "
                  f"{d['sm__warps_active.avg.pct_of_peak_sustained_active']:5.1f}")
    print("per kernel:", ", ".join(f"{k} {v:.0f}" for k, v in sorted(tot.items(), key=lambda x: -x[1])))
    print("total us", round(sum(tot.values()), 1))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 15.0)
