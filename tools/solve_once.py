"""Create the 2-D engine for a config (PCFG, default 4) and run the batched solve twice
(hddm_time_solve): for ncu launch lists of the solve kernels."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1807_04180_b200.problems import config
from paper_1807_04180_b200.engine import DdmEngine
e = DdmEngine(config(int(os.environ.get("PCFG", "4"))))
print("solver", e.solver_desc(), "launches", e.solve_launches())
print("solve ms", e.time_solve(1))
