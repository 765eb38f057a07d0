"""Golden fixture for acceptance criterion a2 (proj/tests/acceptance_tests.cpp:
197-231): the UNMODIFIED reference's global direct solve (direct_solve_global,
oracle.cpp, through oracle/ref_capi.cpp) of the 2x2 protocol problem, stored as
complex64 (the criterion's tolerance is 1e-6 relative).

Run in the build container (needs `make -C oracle ref`):
    python tests/golden/make_golden_a2.py
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_1807_04180_b200.problems import Problem  # noqa: E402
import pyoracle  # noqa: E402


def problem():
    # protocol_grid(200, 2, 2) + constant_medium(freq = 200 / 11) + point_f(0.5, 0.5)
    return Problem("a2_protocol_200_2x2", mx=200, n1=2, n2=2, n_overlap=10, n_ramp=20,
                   omega=2 * math.pi * 200 / 11.0, source=("point", 0.5, 0.5))


if __name__ == "__main__":
    prob = problem()
    u = pyoracle.ref_direct_solve(prob, prob.source_f())
    np.savez_compressed(os.path.join(HERE, "a2_direct.npz"), u=u.astype(np.complex64))
    print("a2 direct solve:", u.shape, float(np.linalg.norm(u)))
