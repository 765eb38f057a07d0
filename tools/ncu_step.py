"""Summarise one DDM step from an ncu --csv launch list (gpu__time_duration +
dram bytes, --print-units base): steps are delimited by k_flags launches; the
last complete step is reported per kernel family, with the solve stage's DRAM
traffic (the roofline `traffic` figure)."""
import collections
import csv
import json
import sys

SOLVE = ("k_ring", "k_fwd_leaf", "k_fwd_pull", "k_fwd_diag", "k_bwd_stage", "k_bwd_pull",
         "k_bwd_diag", "k_bwd_split", "k_bwd_leaf", "k_sep_trsv", "k_fwd_pull_mma",
         "k_fwd_diag_mma", "k_bwd_mma")


def load(path):
    rows = collections.OrderedDict()
    lines = [l for l in open(path) if l.startswith('"')]
    for r in csv.DictReader(lines):
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("hddm::", "").split("<")[0]
        d = rows.setdefault(r["ID"], {"name": name})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "") or 0)
    return list(rows.values())


def main(path, out_json=None):
    ks = load(path)
    starts = [i for i, k in enumerate(ks) if k["name"] == "k_flags"]
    if len(starts) < 2:
        raise SystemExit("need two k_flags launches")
    step = ks[starts[-2]:starts[-1]]
    fam = collections.OrderedDict()
    for k in step:
        f = fam.setdefault(k["name"], [0, 0.0, 0.0])
        f[0] += 1
        f[1] += k["gpu__time_duration.sum"] / 1e3
        f[2] += (k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]) / 1e6
    tot = sum(f[1] for f in fam.values())
    print(f"one step: {len(step)} launches, {tot:.1f} us serialised (ncu, cache flushed per launch)")
    print(f"{'kernel':16s} {'n':>5s} {'us':>9s} {'share':>6s} {'DRAM MB':>9s}")
    for n, (c, us, mb) in sorted(fam.items(), key=lambda x: -x[1][1]):
        print(f"{n:16s} {c:5d} {us:9.1f} {100 * us / tot:5.1f}% {mb:9.1f}")
    solve_us = sum(f[1] for n, f in fam.items() if n in SOLVE)
    solve_mb = sum(f[2] for n, f in fam.items() if n in SOLVE)
    print(f"solve stage: {100 * solve_us / tot:.1f}% of the step, DRAM {solve_mb:.1f} MB per solve")
    if out_json:
        json.dump({"source": path, "launches_per_step": len(step), "step_us_serialised": tot,
                   "solve_share": solve_us / tot, "solve_dram_bytes": solve_mb * 1e6,
                   "families": {n: {"launches": c, "us": us, "dram_mb": mb}
                                for n, (c, us, mb) in fam.items()}},
                  open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
