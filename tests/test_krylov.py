"""The host FGMRES over caller-supplied operators (krylov.py, the reference's
`fgmres(n, A, M, b, x, opt)` API): driven by the C restatement's operators it
must reproduce the restatement's own FGMRES (pinned bit-for-bit to the
reference); driven by the GPU engine's operators it must agree with the
device-resident FGMRES."""
import numpy as np
import pytest

import pyoracle
from conftest import rel_l2
from paper_1807_04180_b200.krylov import FgmresOptions, fgmres
from paper_1807_04180_b200.problems import small


def _dense_system(n, seed):
    rng = np.random.default_rng(seed)
    A = np.eye(n) * 4 + 0.3 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return A, b


def test_small_dense_system_converges():
    A, b = _dense_system(40, 1)
    x, r = fgmres(40, lambda v: A @ v, None, b, FgmresOptions(1e-12, 100, 0))
    assert r.converged and r.true_relres <= 1e-11
    assert np.allclose(x, np.linalg.solve(A, b), rtol=1e-9, atol=1e-12)
    # restarted and preconditioned by a variable operator: still converges
    D = np.diag(1 / np.diag(A))
    k = [0]

    def M(v):
        k[0] += 1
        return (D if k[0] % 2 else np.eye(40)) @ v
    x2, r2 = fgmres(40, lambda v: A @ v, M, b, FgmresOptions(1e-12, 200, 7))
    assert r2.converged and rel_l2(x2, x) <= 1e-9
    # zero right-hand side: x = 0, converged without iterating
    x0, r0 = fgmres(40, lambda v: A @ v, None, np.zeros(40, complex), FgmresOptions())
    assert r0.converged and r0.iters == 0 and not x0.any()


@pytest.mark.parametrize("restart", [0, 3])
def test_matches_restatement_fgmres(restart):
    """Oracle operators in, the oracle's own FGMRES as reference (small config)."""
    prob = small(40, 2, 2, 4.0, 4, 8, source=("gaussian", 0.41, 0.63, 0.02))
    o = pyoracle.OracleEngine(prob)
    f = prob.source_f()
    K = 2
    x, r = fgmres(prob.n_global, o.apply_global, lambda v: o.precondition(v, K), f,
                  FgmresOptions(1e-10, 30, restart))
    xo, ro, _, _ = o.fgmres(f, 1e-10, 30, restart, K)
    assert r.iters == ro.iters and r.converged == ro.converged
    np.testing.assert_allclose(r.history, ro.history, rtol=1e-9, atol=1e-14)
    assert rel_l2(x, xo) <= 1e-9
    assert abs(r.true_relres - ro.true_relres) <= 1e-6 * ro.true_relres + 1e-14


@pytest.mark.gpu
def test_gpu_operators_match_device_fgmres():
    """The reference API driving the GPU operators == the device FGMRES."""
    from paper_1807_04180_b200.engine import DdmEngine, FgmresOptions as DevOpts
    prob = small(80, 2, 2, 8.0, 10, 20, source=("gaussian", 0.41, 0.63, 0.02))
    e = DdmEngine(prob)
    f = prob.source_f()
    K = 2
    x, r = fgmres(prob.n_global, e.apply_global, lambda v: e.precondition(v, K), f,
                  FgmresOptions(1e-8, 40, 30))
    xd, rd = e.fgmres(f, DevOpts(1e-8, 40, 30), K)
    assert r.iters == rd.iters and r.converged == rd.converged
    np.testing.assert_allclose(r.history, rd.history, rtol=1e-7, atol=1e-14)
    assert rel_l2(x, xd) <= 1e-8
    e.close()


def test_reference_krylov_properties():
    """test_krylov.cpp:39-202 re-expressed for the host FGMRES."""
    n = 24
    rng = np.random.default_rng(41)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    # identity: one iteration, exact
    x, r = fgmres(n, lambda v: v.copy(), None, b, FgmresOptions(1e-12, 50, 0))
    assert r.iters == 1 and r.converged and np.allclose(x, b)
    # diagonal: exact within n iterations, true residual recomputed
    d = 1.0 + np.arange(n)
    x, r = fgmres(n, lambda v: d * v, None, b, FgmresOptions(1e-13, n, 0))
    assert r.converged and np.allclose(x, b / d, rtol=1e-11) and r.true_relres <= 1e-12
    # monotone recursive residual, early exit at tol, honest iteration cap
    A = np.eye(n) * 3 + 0.4 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    x, r = fgmres(n, lambda v: A @ v, None, b, FgmresOptions(1e-6, 100, 0))
    assert all(h2 <= h1 * (1 + 1e-12) for h1, h2 in zip(r.history, r.history[1:]))
    assert r.converged and r.relres <= 1e-6 and r.iters == len(r.history)
    x, r = fgmres(n, lambda v: A @ v, None, b, FgmresOptions(1e-15, 5, 0))
    assert r.iters == 5 and not r.converged
    # a variable preconditioner is applied exactly once per iteration
    calls = [0]

    def M(v):
        calls[0] += 1
        return v / np.diag(A) if calls[0] % 2 else v.copy()
    x, r = fgmres(n, lambda v: A @ v, M, b, FgmresOptions(1e-10, 100, 0))
    assert r.converged and calls[0] == r.iters
    # restart still converges; preconditioning helps
    x, r6 = fgmres(n, lambda v: A @ v, None, b, FgmresOptions(1e-10, 200, 6))
    assert r6.converged and r6.true_relres <= 1e-9
    Ainv = np.linalg.inv(A)
    _, rp = fgmres(n, lambda v: A @ v, lambda v: Ainv @ v, b, FgmresOptions(1e-10, 100, 0))
    _, ru = fgmres(n, lambda v: A @ v, None, b, FgmresOptions(1e-10, 100, 0))
    assert rp.iters < ru.iters and rp.iters <= 2
