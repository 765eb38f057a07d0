"""The reference's acceptance criteria a3-a5 (proj/tests/acceptance_tests.cpp:
235-353) on the GPU engine: the criteria themselves, plus the reference's own
step / iteration counts for these problems (recorded by running the reference,
SURVEY.md section 4): a3 4 / 8 / 17 steps, a4 11 / 25 steps, a5 15 / 8 / 1
FGMRES iterations."""
import math

import pytest

from paper_1807_04180_b200.cli import default_layered
from paper_1807_04180_b200.engine import DdmEngine, DdmStats, FgmresOptions
from paper_1807_04180_b200.problems import MEDIUM_LAYERED, Problem

pytestmark = pytest.mark.gpu


def protocol(mx, n, layered=False):
    """protocol_grid + constant_medium / layered_medium, freq = mx / 11
    (acceptance_tests.cpp:64-92); point source at (0.5, 0.5) (point_f)."""
    p = Problem(f"protocol_{mx}_{n}x{n}", mx=mx, n1=n, n2=n, n_overlap=10, n_ramp=20,
                omega=2 * math.pi * mx / 11.0, source=("point", 0.5, 0.5))
    if layered:
        p = p.with_(medium_kind=MEDIUM_LAYERED, layers=default_layered(0.0, 1.0))
    return p


def test_a3_scaling_plateau():
    steps = []
    for mx, n in [(200, 2), (400, 4), (800, 8)]:
        prob = protocol(mx, n)
        with DdmEngine(prob) as e:
            st = DdmStats()
            e.solve_iterative(prob.source_f(), 1e-8, 200, st)
        assert st.converged
        steps.append(st.steps)
    sweeps = [s / (2 * n) for s, n in zip(steps, [2, 4, 8])]
    assert sweeps[2] <= 1.35 * sweeps[1] and sweeps[2] <= 4.0
    assert steps == [4, 8, 17]  # the reference's counts


def test_a4_layered_robustness():
    steps = []
    for n in (2, 4):
        prob = protocol(100 * n, n, layered=True)
        with DdmEngine(prob) as e:
            st = DdmStats()
            e.solve_iterative(prob.source_f(), 1e-8, 400, st)
        assert st.converged
        steps.append(st.steps)
    sweeps = [steps[0] / 4, steps[1] / 8]
    assert max(sweeps) <= 8.0 and sweeps[1] <= 1.5 * sweeps[0]
    assert steps == [11, 25]  # the reference's counts


def test_a5_preconditioner_sweeps():
    prob = protocol(400, 4)
    iters = []
    with DdmEngine(prob) as e:
        f = prob.source_f()
        for K in (1, 2, 8):
            ps = DdmStats()
            x, r = e.fgmres(f, FgmresOptions(1e-8, 300, 0), K, ps)
            assert r.converged and r.true_relres <= 1e-7
            # every preconditioner call visits each window once per sweep
            assert ps.solves + ps.skipped == r.iters * K * prob.nsub
            iters.append(r.iters)
    assert iters[2] * 8 <= iters[0] * 1
    assert iters == [15, 8, 1]  # the reference's counts


def test_a2_four_window_exactness():
    """Point source on both cut lines of a 2x2 split: 4 steps reach relres <=
    1e-3, the converged field deviates <= 1e-6 from the reference's global
    direct solve (tests/golden/a2_direct.npz, make_golden_a2.py); the reference
    converges in 4 steps."""
    import os
    import sys
    import numpy as np
    from conftest import rel_l2
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    from make_golden_a2 import problem
    prob = problem()
    ud = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                              "a2_direct.npz"))["u"].astype(np.complex128)
    with DdmEngine(prob) as e:
        f = prob.source_f()
        st4 = DdmStats()
        e.solve_iterative(f, 0.0, 4, st4)
        assert st4.relres <= 1e-3
        st = DdmStats()
        u = e.solve_iterative(f, 1e-8, 60, st)
    assert st.converged and st.steps == 4
    assert rel_l2(u, ud) <= 1e-6
