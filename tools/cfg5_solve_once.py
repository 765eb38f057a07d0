"""Config 5: create the engine, then 2 batched solves (for ncu launch lists)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1807_04180_b200.problems import config5, small3
from paper_1807_04180_b200.engine3 import DdmEngine3
p = config5() if len(sys.argv) < 2 else small3()
e = DdmEngine3(p)
print("solve launches", e.solve_launches())
print("solve ms", e.time_solve(1))
