"""Phase profile of the dataflow solve (library built with -DHDDM_DAG_PROF, selected
with HDDM_LIB): CTA-cycles per task category and phase over `reps` steady-state
solves of a BASELINE config. Usage: PCFG=4 HDDM_LIB=... python tools/dag_profile.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import dense_residual  # noqa: E402
from paper_1807_04180_b200.engine import DdmEngine, DdmStats  # noqa: E402
from paper_1807_04180_b200.problems import config  # noqa: E402

cfg = int(os.environ.get("PCFG", "4"))
reps = int(os.environ.get("REPS", "10"))
prob = config(cfg)
eng = DdmEngine(prob, device=0)
print(eng.solver_desc(), flush=True)
r = torch.from_numpy(dense_residual(prob)).cuda()
z = torch.empty_like(r)
eng.precondition(r, 3, DdmStats(), out=z)
torch.cuda.synchronize()
eng.dag_profile(reset=True)
ms = eng.time_solve(reps)
p = eng.dag_profile(reset=True)
tot = {k: v for k, v in p.items() if v[6]}
ghz = 1.965e6  # cycles per ms
print(f"solve {ms:.3f} ms; CTA-ms per solve by phase (wait, gather|stage+cols, diag, push|write, ext, "
      "gap to the next task), tasks:")
for k, v in tot.items():
    nrep = reps + 1  # time_solve runs one warm-up launch
    print(f"  {k:16s} " + " ".join(f"{x / ghz / nrep:8.3f}" for x in v[:6]) + f"  tasks {v[6] // nrep}")
print(json.dumps({"cfg": cfg, "solve_ms": ms, "profile": tot}))
import numpy as np  # noqa: E402
tr = eng.dag_trace()
tr = tr[tr[:, 1] > 0]
t0 = tr[:, 0].min()
st, en = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3  # us
span = en.max()
print(f"trace: {len(tr)} tasks over {span:.1f} us, CTAs {len(set(tr[:, 3] % 1000000))}, SMs {len(set(tr[:, 2]))}")
hgt = tr[:, 3] // 1000000
dur = en - st
for kind in (0, 1):
    for d in sorted(set(tr[:, 7])):
        for h in sorted(set(hgt)):
            sel = (tr[:, 4] == kind) & (tr[:, 7] == d) & (hgt == h)
            if sel.any():
                ph = tr[sel][:, 8:12].mean(axis=0) / 1965.0
                print(f"  {'fwd' if kind == 0 else 'bwd'} dec{d} h{h:2d}: {sel.sum():5d} tasks, mean {dur[sel].mean():7.1f} us, "
                      f"max {dur[sel].max():7.1f}, first start {st[sel].min():7.1f}, last end {en[sel].max():7.1f}"
                      f"  phases(us) {' '.join('%.1f' % x for x in ph)}")
grid = np.linspace(0, span, 41)
for a, b in zip(grid[:-1], grid[1:]):
    act = ((st < b) & (en > a))
    fw = act & (tr[:, 4] == 0)
    print(f"  {a:7.1f}-{b:7.1f} us: active {act.sum():5d} (fwd {fw.sum():5d})  started {((st >= a) & (st < b)).sum():5d}")
np.save("gpurun_out/dag_trace.npy", tr)
