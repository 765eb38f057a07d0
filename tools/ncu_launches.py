"""Driver for an ncu launch list of DDM steps (run under ncu; graphs off so every kernel
is its own launch): one engine, `PSTEPS` sweeps of precondition on a dense seeded residual.
    HDDM_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,\\
        dram__bytes_write.sum --clock-control none --csv --print-units base \\
        --log-file launches.csv python tools/ncu_launches.py 4
then `python tools/ncu_step.py launches.csv summary.json` (the last complete step)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import dense_residual  # noqa: E402
from paper_1807_04180_b200.engine import DdmEngine, DdmStats  # noqa: E402
from paper_1807_04180_b200.problems import config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prob = config(cfg)
with DdmEngine(prob) as e:
    e.precondition(dense_residual(prob), int(os.environ.get("PSTEPS", "4")), DdmStats())
