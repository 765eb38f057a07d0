"""Time the batched solve stage alone (hddm_time_solve: the solve graph of one
DDM step's right-hand sides, CUDA events on the engine stream) for a BASELINE
config. Profiling knobs (read by the engine, results of the solve invalid when
set): HDDM_TIME_SPARSE=1 (steady-state forward plan), HDDM_SKIP=<mask> (leave
kernel families out), HDDM_ONLY_M=<M> / HDDM_ONLY_TILE=<g> (one kind of tile
group), HDDM_TIME_EMPTY=1 (launch/dependency floor), HDDM_TIME_PAIR=1 (two
solve graphs concurrently). Usage: PCFG=4 python tools/time_solve.py"""
import os, sys, json, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1807_04180_b200.engine import DdmEngine, DdmStats
from paper_1807_04180_b200.problems import config
from bench import dense_residual
cfg = int(os.environ.get("PCFG", "4"))
prob = config(cfg)
t0 = time.time()
eng = DdmEngine(prob, device=0)
t1 = time.time()
r = torch.from_numpy(dense_residual(prob)).cuda()
z = torch.empty_like(r)
eng.precondition(r, 3, DdmStats(), out=z)
torch.cuda.synchronize()
ms = [eng.time_solve(20) for _ in range(3)]
tag = os.environ.get("TAG", "")
print(f"RESULT {tag} solve_ms={min(ms):.4f} all={['%.4f'%m for m in ms]} create_s={t1-t0:.1f}", flush=True)
