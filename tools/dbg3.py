"""3-D engine vs the 3-D restatement on small cases (debug driver)."""
import sys, os, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
from paper_1807_04180_b200.problems import small3
from paper_1807_04180_b200.engine3 import DdmEngine3
from paper_1807_04180_b200.engine import DdmStats, FgmresOptions
import pyoracle

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

for p in [small3(), small3(m=24, n=4, freq=2.0, n_ov=2, n_ramp=2)]:
    t = time.time(); e = DdmEngine3(p); t1 = time.time() - t
    o = pyoracle.Oracle3Engine(p)
    print(p.name, "create", round(t1, 2), "s factor_ms", e.factor_ms(), "classes", len(e.class_info()))
    ci, oi = e.class_info(), o.class_info()
    print(" members eq", [c["members"] for c in ci] == [c["members"] for c in oi],
          "nnz eq", ci[0]["factor_nnz"] == oi[0]["factor_nnz"],
          "probe max", max(c["probe_relres"] for c in ci))
    nw = int(np.prod(e.window_dims()))
    rng = np.random.default_rng(0)
    b = rng.standard_normal(nw) + 1j * rng.standard_normal(nw)
    for c in range(min(3, len(ci))):
        xg, rg = e.class_solve(c, b)
        xo, ro = o.class_solve(c, b)
        print("  class", c, "solve rel", rel(xg, xo), "relres", rg, ro)
    f = p.source_f()
    u = rng.standard_normal(p.n_global) + 1j * rng.standard_normal(p.n_global)
    print(" apply rel", rel(e.apply_global(u), o.apply_global(u)))
    for K in (1, 2, 3, 4):
        st = DdmStats()
        zg = e.precondition(f, K, st)
        zo = o.precondition(f, K, None)
        print("  precond K", K, "rel", rel(zg, zo), "solves", st.solves, st.skipped, "refine", e.refine_stats())
    x, r = e.fgmres(f, FgmresOptions(1e-6, 100, 30), p.k_steps)
    xo, ro, ps, _ = o.fgmres(f, 1e-6, 100, 30, p.k_steps)
    print(" fgmres iters", r.iters, ro.iters, "x rel", rel(x, xo), "true relres", r.true_relres, ro.true_relres)
    e.close()
