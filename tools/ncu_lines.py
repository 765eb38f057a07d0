"""Attribute ncu warp-stall samples (SASS source page) to CUDA source lines.

usage: ncu_lines.py REPORT.ncu-rep KERNEL_REGEX LIB.so FUNC_SUBSTR [top]
Extracts the cubins from LIB.so, maps SASS offsets to lines with `nvdisasm -g`,
and sums the samples of the profiled kernel per source line."""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile


def line_map(lib, func_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        m = None
        for sec in txt.split("//--------------------- .text."):
            if sec.startswith(func_sub) or func_sub in sec.split(" ")[0]:
                m = sec
                break
        if m is None:
            continue
        cur = None
        out = {}
        for ln in m.splitlines():
            g = re.search(r'File "([^"]+)", line (\d+)', ln) if "//## File" in ln else None
            if g:
                cur = (g.group(1), int(g.group(2)))
                continue
            a = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
            if a and cur is not None:
                out[int(a.group(1), 16)] = cur
        return out
    raise SystemExit("function not found")


def samples(rep, kregex):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kregex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = None
    out = []
    done = []
    for r in rows:
        if r and r[0] == "Address":  # one table per launch: all matching launches are summed
            hdr = {k: i for i, k in enumerate(r)}
            if out:
                base0 = min(a for a, _, _ in out)
                done.extend((a - base0, s_, n) for a, s_, n in out)
                out = []
            continue
        if hdr and len(r) >= len(hdr):
            out.append((int(r[hdr["Address"]], 16), float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0),
                        float(r[hdr["Instructions Executed"]] or 0)))
    base = min(a for a, _, _ in out)
    return done + [(a - base, s, n) for a, s, n in out]


def main():
    rep, kre, lib, fsub = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
    lm = line_map(lib, fsub)
    files = {}
    acc = collections.Counter()
    ins = collections.Counter()
    for off, s, n in samples(rep, kre):
        acc[lm.get(off, ("?", 0))] += s
        ins[lm.get(off, ("?", 0))] += n
    tot = sum(acc.values())
    itot = sum(ins.values()) or 1
    print(f"warp instructions executed: {itot:.0f}")
    for (fn, ln), s in acc.most_common(top):
        if fn not in files:
            files[fn] = open(fn).read().splitlines() if os.path.exists(fn) else []
        src = files[fn]
        text = src[ln - 1].strip()[:90] if 0 < ln <= len(src) else ""
        print(f"{100 * s / tot:5.1f}% stall {100 * ins[(fn, ln)] / itot:5.1f}% inst  {os.path.basename(fn)}:{ln:<5d} {text}")


if __name__ == "__main__":
    main()
