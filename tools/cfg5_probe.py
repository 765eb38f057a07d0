"""Config 5 (3-D) on the GPU: factorization, solve-stage time, a K=6 precondition and the
FGMRES(30)+DDM(6) solve (measurement driver)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1807_04180_b200.problems import config5
from paper_1807_04180_b200.engine3 import DdmEngine3, symbolic_stats3
from paper_1807_04180_b200.engine import DdmStats, FgmresOptions
from paper_1807_04180_b200.roofline import step_bytes3

p = config5()
print("window", p.window, "n_global", p.n_global, symbolic_stats3(*p.window), flush=True)
t = time.time()
e = DdmEngine3(p)
print("create s", time.time() - t, "factor_ms", e.factor_ms(), "footprint", e.footprint(), flush=True)
ci = e.class_info()
print("classes", len(ci), "probe max", max(c["probe_relres"] for c in ci), flush=True)
f = p.source_f()
r = torch.from_numpy(f).cuda()
z = torch.empty_like(r)
st = DdmStats()
e.precondition(r, 6, st, out=z)
torch.cuda.synchronize()
t = time.time()
st = DdmStats()
e.precondition(r, 6, st, out=z)
torch.cuda.synchronize()
dt = time.time() - t
print("precondition K=6 wall ms", 1e3 * dt, "per step", 1e3 * dt / 6, "solves", st.solves, st.skipped,
      "refine", e.refine_stats(), flush=True)
ms = e.time_solve(10)
B = step_bytes3(p, [c["factor_nnz"] for c in ci])
print("solve ms", ms, "B_solve GB", B["B_solve"] / 1e9, "GB/s", B["B_solve"] / (ms / 1e3) / 1e9, flush=True)
x, res = e.fgmres(f, FgmresOptions(1e-6, 200, 30), 6)
t = time.time()
x, res = e.fgmres(f, FgmresOptions(1e-6, 200, 30), 6)
dt = time.time() - t
print("fgmres iters", res.iters, "true relres", res.true_relres, "wall s", dt, "hist", res.history, flush=True)
print("refine", e.refine_stats())
