"""Coordinate-descent tuner for the lane shapes of the steady-state forward
levels (hddm_tune_fwd_shape): for each table (0/1 pulls of singleton / member
tiles, 2/3 inverse rows) and level, try every valid E and keep the fastest DDM
step (precondition(r, K=32), CUDA events). Prints the tables as the environment
strings HDDM_FWDP_E1 / HDDM_FWDP_EM / HDDM_FWDD_E1 / HDDM_FWDD_EM.
Usage: PCFG=4 python tools/tune_fwd_shapes.py [passes]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import dense_residual  # noqa: E402
from paper_1807_04180_b200.engine import DdmEngine, DdmStats  # noqa: E402
from paper_1807_04180_b200.problems import config  # noqa: E402

prob = config(int(os.environ.get("PCFG", "4")))
eng = DdmEngine(prob, device=0)
members = max(c["members"] for c in eng.class_info())
mtile = min(16, members)
r = torch.from_numpy(dense_residual(prob)).cuda()
z = torch.empty_like(r)
stream = torch.cuda.ExternalStream(eng.stream_handle(), device="cuda:0")
NLEV = int(os.environ.get("NLEV", "12"))


def measure():
    eng.precondition(r, 2, DdmStats(), out=z)
    best = 1e9
    for _ in range(2):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.precondition(r, 32, DdmStats(), out=z)
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 32)
    return best


tab = {w: [0] * NLEV for w in range(4)}
best = measure()
print(f"start {best:.4f} ms/step", flush=True)
passes = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for p in range(passes):
    for w in (1, 3, 0, 2):
        M = mtile if w in (1, 3) else 1
        cands = [e for e in (0, 1, 2, 4, 8, 16, 32) if e * M <= 32]
        for lev in range(NLEV):
            keep = tab[w][lev]
            for e in cands:
                if e == keep:
                    continue
                eng.tune_fwd_shape(w, lev, e)
                t = measure()
                if t < best * 0.997:
                    best, keep = t, e
                    print(f"  table {w} level {lev}: E={e} -> {best:.4f}", flush=True)
            eng.tune_fwd_shape(w, lev, keep)
            tab[w][lev] = keep
    print(f"pass {p}: {best:.4f} ms/step", flush=True)
names = ["HDDM_FWDP_E1", "HDDM_FWDP_EM", "HDDM_FWDD_E1", "HDDM_FWDD_EM"]
print("RESULT " + " ".join(f"{names[w]}={','.join(map(str, tab[w]))}" for w in range(4)), flush=True)
eng.close()
