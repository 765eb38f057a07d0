"""Algorithmic byte counts of one DDM iteration.

B_step = B_fac + B_vec + B_xfer + B_acc (+ B_res standalone), index arrays
excluded:

* B_fac  = sum over classes with >= 1 active member of 16 (2 nnzL_c + n_w):
           every distinct factor read once for the forward and once for the
           backward sweep (nnzL_c = factor_nonzeros() - n_w, sparse.cpp:238-240);
* B_vec  = sum over active subdomains of 2 * 16 * n_w (rhs in, solution out);
* B_xfer = sum over executed (target, direction) of 16 (|patch| + |w buffer|)
           (transfer.cpp:7-88);
* B_acc  = sum over active subdomains of 48 |blend region| (ddm.cpp:216-235);
* B_res  = 40 N_g (u, f, k^2; residual_norm, ddm.cpp:237-242).

The solve stage (the dominant kernel group) is charged B_fac + B_vec.
"""
from __future__ import annotations

from typing import Dict

from .problems import Problem

_DI = (+1, -1, 0, 0, +1, -1, +1, -1)
_DJ = (0, 0, +1, -1, +1, +1, -1, -1)


def _geometry(p: Problem):
    ext = p.n_ext
    mcx, mcy = p.mx // p.n1, p.my // p.n2
    wnx, wny = p.window
    subs = []
    for j in range(p.n2):
        for i in range(p.n1):
            cx0 = ext + i * mcx
            cy0 = ext + j * mcy
            subs.append(dict(i=i, j=j, cx0=cx0, cx1=cx0 + mcx, cy0=cy0, cy1=cy0 + mcy,
                             wx0=cx0 - ext, wy0=cy0 - ext))
    return subs, wnx, wny


def _patch(d: int, s: dict, wnx: int, wny: int, nov: int):
    p0, p1 = s["wx0"] + 1, s["wx0"] + wnx - 2
    q0, q1 = s["wy0"] + 1, s["wy0"] + wny - 2
    from_l = d in (1, 5, 7)
    from_r = d in (0, 4, 6)
    from_b = d in (3, 6, 7)
    from_t = d in (2, 4, 5)
    if from_l:
        p0, p1 = max(p0, s["cx0"] + 1), min(p1, s["cx0"] + 1 + nov)
    if from_r:
        p0, p1 = max(p0, s["cx1"] - 1 - nov), min(p1, s["cx1"] - 1)
    if from_b:
        q0, q1 = max(q0, s["cy0"] + 1), min(q1, s["cy0"] + 1 + nov)
    if from_t:
        q0, q1 = max(q0, s["cy1"] - 1 - nov), min(q1, s["cy1"] - 1)
    return p0, p1, q0, q1


def step_bytes(p: Problem, nnz_per_class, members_per_class, standalone: bool = False
               ) -> Dict[str, float]:
    """Steady-state bytes of one DDM iteration with every subdomain active."""
    subs, wnx, wny = _geometry(p)
    nw = wnx * wny
    b_fac = sum(16.0 * (2.0 * (nnz - nw) + nw) for nnz in nnz_per_class)
    b_vec = 2.0 * 16.0 * nw * len(subs)
    b_xfer = 0.0
    b_acc = 0.0
    for s in subs:
        for d in range(8):
            si, sj = s["i"] + _DI[d], s["j"] + _DJ[d]
            if not (0 <= si < p.n1 and 0 <= sj < p.n2):
                continue
            p0, p1, q0, q1 = _patch(d, s, wnx, wny, p.n_overlap)
            if p1 < p0 or q1 < q0:
                continue
            patch = (p1 - p0 + 1) * (q1 - q0 + 1)
            wbuf = (p1 - p0 + 3) * (q1 - q0 + 3)
            b_xfer += 16.0 * (patch + wbuf)
        x0 = s["cx0"] - p.n_overlap if s["i"] > 0 else s["wx0"]
        x1 = s["cx1"] + p.n_overlap if s["i"] < p.n1 - 1 else s["wx0"] + wnx - 1
        y0 = s["cy0"] - p.n_overlap if s["j"] > 0 else s["wy0"]
        y1 = s["cy1"] + p.n_overlap if s["j"] < p.n2 - 1 else s["wy0"] + wny - 1
        b_acc += 48.0 * (x1 - x0 + 1) * (y1 - y0 + 1)
    b_res = 40.0 * p.n_global if standalone else 0.0
    out = dict(B_fac=b_fac, B_vec=b_vec, B_xfer=b_xfer, B_acc=b_acc, B_res=b_res)
    out["B_solve"] = b_fac + b_vec
    out["B_step"] = b_fac + b_vec + b_xfer + b_acc + b_res
    return out


def step_bytes3(p, nnz_per_class) -> Dict[str, float]:
    """The same count for a 3-D problem (Problem3, config 5): 26 transfer
    directions (hddm_oracle3.c transfer_patch3), box blend regions."""
    ext, nov = p.n_ext, p.n_overlap
    nd = (p.n1, p.n2, p.n3)
    mc = (p.mx // p.n1, p.my // p.n2, p.mz // p.n3)
    nn = p.window
    nw = nn[0] * nn[1] * nn[2]
    nsub = p.nsub
    b_fac = sum(16.0 * (2.0 * (nnz - nw) + nw) for nnz in nnz_per_class)
    b_vec = 2.0 * 16.0 * nw * nsub
    dirs = [(a, b, c) for c in (-1, 0, 1) for b in (-1, 0, 1) for a in (-1, 0, 1) if (a, b, c) != (0, 0, 0)]
    b_xfer = b_acc = 0.0
    for t in range(nsub):
        ix = (t % nd[0], (t // nd[0]) % nd[1], t // (nd[0] * nd[1]))
        c0 = [ext + ix[a] * mc[a] for a in range(3)]
        c1 = [c0[a] + mc[a] for a in range(3)]
        w0 = [c0[a] - ext for a in range(3)]
        for o in dirs:
            if not all(0 <= ix[a] + o[a] < nd[a] for a in range(3)):
                continue
            vol = wvol = 1
            for a in range(3):
                lo, hi = w0[a] + 1, w0[a] + nn[a] - 2
                if o[a] > 0:
                    lo, hi = max(lo, c1[a] - 1 - nov), min(hi, c1[a] - 1)
                elif o[a] < 0:
                    lo, hi = max(lo, c0[a] + 1), min(hi, c0[a] + 1 + nov)
                vol *= max(0, hi - lo + 1)
                wvol *= max(0, hi - lo + 3)
            if vol:
                b_xfer += 16.0 * (vol + wvol)
        reg = 1
        for a in range(3):
            x0 = c0[a] - nov if ix[a] > 0 else w0[a]
            x1 = c1[a] + nov if ix[a] < nd[a] - 1 else w0[a] + nn[a] - 1
            reg *= x1 - x0 + 1
        b_acc += 48.0 * reg
    out = dict(B_fac=b_fac, B_vec=b_vec, B_xfer=b_xfer, B_acc=b_acc, B_res=0.0)
    out["B_solve"] = b_fac + b_vec
    out["B_step"] = b_fac + b_vec + b_xfer + b_acc
    return out
