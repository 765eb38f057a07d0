"""The device-resident FGMRES (hddm_fgmres: one CUDA graph per restart cycle, state in
HBM) against the C restatement's FGMRES (pinned bit-for-bit to the reference,
krylov.cpp:24-133) on the same operators, and the reference's Krylov properties
(test_krylov.cpp) that apply to A = apply_global, M = precondition(K).

Host-lambda callers (any A / M) use the reference's OWN fgmres: the drop-in build of
the reference (tests/test_dropin.py) drives the GPU engine through it."""
import numpy as np
import pytest

import pyoracle
from conftest import rel_l2
from paper_1807_04180_b200.problems import small

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    from paper_1807_04180_b200.engine import DdmEngine
    prob = small(40, 2, 2, 4.0, 4, 8, source=("gaussian", 0.41, 0.63, 0.02))
    e = DdmEngine(prob)
    o = pyoracle.OracleEngine(prob)
    yield prob, e, o
    e.close()
    o.close()


@pytest.mark.parametrize("restart", [0, 3, 30])
def test_device_fgmres_matches_restatement(pair, restart):
    """Same iterations, recursive residual history, solution and true residual as the
    restatement's FGMRES; restarts (the explicit residual recompute) included."""
    from paper_1807_04180_b200.engine import DdmStats, FgmresOptions
    prob, e, o = pair
    f = prob.source_f()
    K = 2
    ps = DdmStats()
    x, r = e.fgmres(f, FgmresOptions(1e-10, 30, restart), K, ps)
    xo, ro, pso, _ = o.fgmres(f, 1e-10, 30, restart, K)
    assert r.iters == ro.iters and r.converged == ro.converged
    np.testing.assert_allclose(r.history, ro.history, rtol=1e-6, atol=1e-13)
    assert rel_l2(x, xo) <= 1e-9
    assert abs(r.true_relres - ro.true_relres) <= 1e-6 * ro.true_relres + 1e-14
    assert (ps.solves, ps.skipped) == (pso.solves, pso.skipped)


def test_device_fgmres_properties(pair):
    """test_krylov.cpp's properties on the device FGMRES: zero right-hand side returns
    x = 0 converged without iterating; the recursive residual is monotone; an honest
    iteration cap; one preconditioner application (K sweeps of every subdomain) per
    iteration."""
    from paper_1807_04180_b200.engine import DdmStats, FgmresOptions
    prob, e, o = pair
    x0, r0 = e.fgmres(np.zeros(prob.n_global, complex), FgmresOptions(1e-8, 20, 0), 2)
    assert r0.converged and r0.iters == 0 and not np.any(x0)
    f = prob.source_f()
    ps = DdmStats()
    _, r = e.fgmres(f, FgmresOptions(1e-30, 4, 0), 1, ps)
    assert all(h2 <= h1 * (1 + 1e-12) for h1, h2 in zip(r.history, r.history[1:]))
    assert r.iters == len(r.history) == 4 and not r.converged and np.isfinite(r.true_relres)
    assert ps.solves + ps.skipped == r.iters * 1 * prob.nsub
    # restarted still converges
    _, r5 = e.fgmres(f, FgmresOptions(1e-9, 200, 5), 2)
    assert r5.converged and r5.true_relres <= 2e-9
