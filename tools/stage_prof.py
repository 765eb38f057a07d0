"""Stage kernels of one DDM step timed alone (hddm_time_kernel: transfer, residual check,
blend-accumulate on the last sweep's state) for a BASELINE config; under ncu, REPS=1 keeps
the launch list short. Usage: PCFG=4 [REPS=20] python tools/stage_prof.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1807_04180_b200.engine import DdmEngine, DdmStats
from paper_1807_04180_b200.problems import config
from bench import dense_residual
prob = config(int(os.environ.get("PCFG", "4")))
eng = DdmEngine(prob, device=0)
r = torch.from_numpy(dense_residual(prob)).cuda()
z = torch.empty_like(r)
eng.precondition(r, 4, DdmStats(), out=z)
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", "20"))
for k in ("transfer", "check", "accumulate"):
    print(f"STAGE {os.environ.get('TAG','')} {k} ms={eng.time_kernel(k, reps):.4f}", flush=True)
