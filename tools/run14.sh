python tools/cfg5_solve_once.py 2>&1 | grep "solve ms"
HDDM3_PDL=1 python tools/cfg5_solve_once.py 2>&1 | grep "solve ms"
python -c "
import sys; sys.path.insert(0,'.')
from paper_1807_04180_b200.problems import config5
from paper_1807_04180_b200.engine3 import DdmEngine3
e=DdmEngine3(config5()); print('plain', [round(e.time_solve(20),3) for _ in range(3)])"
HDDM3_PDL=1 python -c "
import sys; sys.path.insert(0,'.')
from paper_1807_04180_b200.problems import config5
from paper_1807_04180_b200.engine3 import DdmEngine3
e=DdmEngine3(config5()); print('pdl', [round(e.time_solve(20),3) for _ in range(3)])"
HDDM3_PDL=1 python -m pytest tests/test_gpu_3d.py -x -q 2>&1 | tail -2
