python -c "
import sys; sys.path.insert(0,'.')
from paper_1807_04180_b200.problems import config5
from paper_1807_04180_b200.engine3 import DdmEngine3
e=DdmEngine3(config5()); print('solve', [round(e.time_solve(20),3) for _ in range(3)], 'launches', e.solve_launches())"
python -m pytest tests/test_gpu_3d.py -x -q 2>&1 | tail -2
