"""Key metrics of an `ncu --set full` report (details page) plus the top SASS
stall lines: python tools/ncu_full_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Grid Size", "Block Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "Warp Cycles Per Issued Instruction", "Theoretical Occupancy",
        "Achieved Occupancy", "Avg. Active Threads Per Warp"]


def main(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    seen = set()
    for r in csv.reader(io.StringIO(det)):
        if len(r) > 14 and r[12] in WANT and r[12] not in seen:
            seen.add(r[12])
            if len(seen) == 1:
                print(f"kernel: {r[4][:100]}")
            print(f"  {r[12]:40s} {r[14]:>14s} {r[13]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "Address":
            hdr = {k: i for i, k in enumerate(r)}
            continue
        if hdr and len(r) >= len(hdr):
            s = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
            out.append((s, r[hdr["Source"]].strip()))
    tot = sum(s for s, _ in out) or 1
    print("  top stall-sampled SASS:")
    for s, src_line in sorted(out, key=lambda x: -x[0])[:10]:
        print(f"    {100 * s / tot:5.1f}%  {src_line[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])
