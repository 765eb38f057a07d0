"""Config 5 factorization time (DMMA trailing updates by default; HDDM3_FACTOR_FMA=1:
CUDA-core FMA kernel) and the probe residuals."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1807_04180_b200.problems import config5
from paper_1807_04180_b200.engine3 import DdmEngine3
e = DdmEngine3(config5())
ci = e.class_info()
print(f"RESULT fma={os.environ.get('HDDM3_FACTOR_FMA','0')} factor_ms={e.factor_ms():.1f} "
      f"probe_max={max(c['probe_relres'] for c in ci):.3e}", flush=True)
