"""Time DDM steps (one precondition(r, K=32) call, CUDA events, like bench.py's
`value`) for a BASELINE config. Profiling knobs: HDDM_STEP_NOSOLVE=1 (everything
but the solve), HDDM_STEP_SKIP=<mask> (1 flags, 2 gather, 4 check, 8 accumulate;
results invalid). Usage: PCFG=4 python tools/time_step.py"""
import os, sys, time
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
stream = torch.cuda.ExternalStream(eng.stream_handle(), device="cuda:0")
eng.precondition(r, 3, DdmStats(), out=z)
torch.cuda.synchronize()
K = 32
res = []
for rep in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    eng.precondition(r, K, DdmStats(), out=z)
    e1.record(stream)
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / K)
print(f"RESULT {os.environ.get('TAG','')} ms_per_step={min(res):.4f} all={['%.4f'%x for x in res]}", flush=True)
