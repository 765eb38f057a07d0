"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    out = []
    kernel = None
    hdr = None
    for r in rows:
        if r and r[0] == "Kernel Name":
            kernel = r[1]
            continue
        if r and r[0] == "Address":
            hdr = {k: i for i, k in enumerate(r)}
            continue
        if hdr and len(r) >= len(hdr):
            s = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
            out.append((s, kernel, r[hdr["Address"]][-5:], r[hdr["Source"]].strip()))
    tot = {}
    for s, k, a, src in out:
        tot[k] = tot.get(k, 0) + s
    for k, t in tot.items():
        print(f"== {k[:90]}  total samples {t:.0f}")
        items = sorted([o for o in out if o[1] == k], key=lambda o: -o[0])[:top]
        for s, _, a, src in items:
            print(f"  {100 * s / t:5.1f}%  {a}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
