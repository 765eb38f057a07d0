"""The 3-D path (BASELINE config 5, include/hddm3.h) on the GPU against the 3-D
restatement (oracle/hddm_oracle3.c) on identical inputs, through the C-ABI.

Parity is against the restatement only: the reference has no 3-D code (its
parity is unpinned). The restatement itself is checked
against a numpy operator and a direct global solve (tests/test_oracle3.py).
Tolerances are north_star's: per-iteration iterates <= 1e-10 relative L2, final
solution <= 1e-8, identical solve / skip / FGMRES iteration counts."""
import math

import numpy as np
import pytest

import pyoracle
from conftest import rel_l2
from paper_1807_04180_b200.problems import config5, small3

pytestmark = pytest.mark.gpu

CASES = {
    "2x2x2": small3(m=16, n=2, freq=3.0, n_ov=2, n_ramp=3),
    "4x4x4": small3(m=24, n=4, freq=2.0, n_ov=2, n_ramp=2,
                    source=("gaussian", 0.3, 0.62, 0.41, 0.1)),
    "3x2x2": small3(m=18, n=2, freq=2.5, n_ov=2, n_ramp=3).with_(n1=3, mx=18, my=16, mz=16,
                                                                  h=1.0 / 18),
}


@pytest.fixture(scope="module", params=list(CASES))
def pair(request):
    from paper_1807_04180_b200.engine3 import DdmEngine3
    prob = CASES[request.param]
    e = DdmEngine3(prob)
    o = pyoracle.Oracle3Engine(prob)
    yield prob, e, o
    e.close()
    o.close()


def test_setup_matches_restatement(pair):
    prob, e, o = pair
    ci, oi = e.class_info(), o.class_info()
    assert [c["members"] for c in ci] == [c["members"] for c in oi]
    assert [e.class_of(t) for t in range(prob.nsub)] == [o.class_of(t) for t in range(prob.nsub)]
    assert [c["factor_nnz"] for c in ci] == [c["factor_nnz"] for c in oi]
    assert all(c["probe_relres"] <= 1e-12 for c in ci)
    assert abs(e.sigma0() - o.sigma0) <= 1e-14 * o.sigma0
    assert e.n_global() == prob.n_global


def test_class_solves_match(pair):
    prob, e, o = pair
    nw = int(np.prod(prob.window))
    rng = np.random.default_rng(7)
    b = rng.standard_normal(nw) + 1j * rng.standard_normal(nw)
    for c in range(len(e.class_info())):
        xg, rg = e.class_solve(c, b)
        xo, _ = o.class_solve(c, b)
        assert rel_l2(xg, xo) <= 1e-12
        assert rg <= 1e-11
        r = b - o.class_matvec(c, xg)  # the restatement's assembled matrix
        assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-11


def test_apply_global_matches(pair):
    prob, e, o = pair
    rng = np.random.default_rng(3)
    u = rng.standard_normal(prob.n_global) + 1j * rng.standard_normal(prob.n_global)
    assert rel_l2(e.apply_global(u), o.apply_global(u)) <= 1e-14


def test_per_step_iterates_and_counts(pair):
    from paper_1807_04180_b200.engine import DdmStats
    prob, e, o = pair
    f = prob.source_f()
    for K in range(1, prob.k_steps + 2):
        st, so = DdmStats(), pyoracle.Stats()
        zg = e.precondition(f, K, st)
        zo = o.precondition(f, K, so)
        assert rel_l2(zg, zo) <= 1e-10, K
        assert (st.solves, st.skipped) == (so.solves, so.skipped), K


def test_subdomain_taps_match(pair):
    prob, e, o = pair
    f = prob.source_f()
    e.precondition(f, 2)
    o.precondition(f, 2)
    for t in range(prob.nsub):
        rg, ug, ag = e.tap_subdomain(t)
        ro, uo, ao = o.tap_subdomain(t)
        assert ag == ao
        if ao:
            assert rel_l2(rg, ro) <= 1e-12
            assert rel_l2(ug, uo) <= 1e-10


def test_solve_iterative_matches(pair):
    from paper_1807_04180_b200.engine import DdmStats
    prob, e, o = pair
    f = prob.source_f()
    st = DdmStats()
    u = e.solve_iterative(f, 0.0, 5, st)
    uo, so = o.solve_iterative(f, 0.0, 5)
    assert rel_l2(u, uo) <= 1e-10
    assert (st.steps, st.solves, st.skipped) == (so.steps, so.solves, so.skipped)
    assert np.allclose([h.relres for h in st.history], [h[1] for h in so.history], rtol=1e-8)


def test_fgmres_matches(pair):
    from paper_1807_04180_b200.engine import DdmStats, FgmresOptions
    prob, e, o = pair
    f = prob.source_f()
    ps = DdmStats()
    x, res = e.fgmres(f, FgmresOptions(1e-6, 40, 30), prob.k_steps, ps)
    xo, ro, pso, zo = o.fgmres(f, 1e-6, 40, 30, prob.k_steps, keep_z=2)
    assert res.iters == ro.iters and res.converged == ro.converged
    assert rel_l2(x, xo) <= 1e-8
    assert np.allclose(res.history, ro.history, rtol=1e-6)
    assert (ps.solves, ps.skipped) == (pso.solves, pso.skipped)


def test_zero_scaling_determinism(pair):
    prob, e, o = pair
    f = prob.source_f()
    z1 = e.precondition(f, 3)
    assert np.array_equal(e.precondition(2.0 * f, 3), 2.0 * z1)  # exact: powers of two
    assert np.array_equal(e.precondition(f, 3), z1)               # deterministic
    assert not e.precondition(np.zeros_like(f), 3).any()


def test_point_source_causality():
    """One subdomain holds the source: a subdomain at Manhattan distance d first
    solves at step d + 1 (faces s-1, edges s-2, vertices s-3 all advance one axis
    per step), exactly as the restatement's skip rules say."""
    from paper_1807_04180_b200.engine import DdmStats
    from paper_1807_04180_b200.engine3 import DdmEngine3
    prob = small3(m=18, n=3, freq=2.0, n_ov=2, n_ramp=2, source=("point", 0.1, 0.12, 0.15))
    e = DdmEngine3(prob)
    o = pyoracle.Oracle3Engine(prob)
    f = prob.source_f()
    for K in range(1, 8):
        st, so = DdmStats(), pyoracle.Stats()
        zg = e.precondition(f, K, st)
        zo = o.precondition(f, K, so)
        assert (st.solves, st.skipped) == (so.solves, so.skipped)
        assert rel_l2(zg, zo) <= 1e-10
    st = DdmStats()
    e.precondition(f, 1, st)
    assert (st.solves, st.skipped) == (1, 26)
    e.close()


def test_device_memory_path(pair):
    import torch
    prob, e, o = pair
    f = prob.source_f()
    ft = torch.from_numpy(f).cuda()
    zt = e.precondition(ft, 2)
    assert rel_l2(zt.cpu().numpy(), e.precondition(f, 2)) == 0.0


# ------------------------------------------------------------- config 5 at full size
def _alpha(m, c0, c1, lo, hi, prob, sigma0):
    h2, d = 0.5 * prob.h, prob.n_ramp * prob.h

    def shifted(t, dsh):
        t = np.asarray(t, float)
        s = np.clip((t - dsh) / d, 0.0, 1.0)
        return np.where(t <= dsh, 0.0, np.where(t >= dsh + d, sigma0, sigma0 * s * s))
    m = np.asarray(m)
    sig = np.where(2 * c0 - m > 0, shifted((2 * c0 - m) * h2, prob.n_overlap * prob.h if lo else 0.0), 0.0)
    sig = sig + np.where(m - 2 * c1 > 0, shifted((m - 2 * c1) * h2, prob.n_overlap * prob.h if hi else 0.0), 0.0)
    return 1.0 + 1j * sig


def _global_apply_numpy(prob, sigma0, u):
    """Vectorized L-form 3-D operator (identity on the shell): an independent
    restatement of the formulas for full-size checks."""
    gx, gy, gz = prob.gdims
    e = prob.n_ext
    ms = (prob.mx, prob.my, prob.mz)
    an = [_alpha(2 * np.arange(n), e, e + ms[a], 0, 0, prob, sigma0) for a, n in enumerate((gx, gy, gz))]
    ia = [1.0 / _alpha(2 * np.arange(n) + 1, e, e + ms[a], 0, 0, prob, sigma0) for a, n in enumerate((gx, gy, gz))]
    U = u.reshape(gz, gy, gx)
    out = U.copy()
    k2 = (prob.omega / prob.velocity) ** 2
    ih2 = 1.0 / prob.h ** 2
    a1, a2, a3 = an[0][None, None, 1:-1], an[1][None, 1:-1, None], an[2][1:-1, None, None]
    i1p, i1m = ia[0][None, None, 1:-1], ia[0][None, None, :-2]
    i2p, i2m = ia[1][None, 1:-1, None], ia[1][None, :-2, None]
    i3p, i3m = ia[2][1:-1, None, None], ia[2][:-2, None, None]
    c = U[1:-1, 1:-1, 1:-1]
    t = (a2 * a3 * ih2) * (i1p * (U[1:-1, 1:-1, 2:] - c) - i1m * (c - U[1:-1, 1:-1, :-2])) \
        + (a1 * a3 * ih2) * (i2p * (U[1:-1, 2:, 1:-1] - c) - i2m * (c - U[1:-1, :-2, 1:-1])) \
        + (a1 * a2 * ih2) * (i3p * (U[2:, 1:-1, 1:-1] - c) - i3m * (c - U[:-2, 1:-1, 1:-1]))
    out[1:-1, 1:-1, 1:-1] = t / (a1 * a2 * a3) + k2 * c
    return out.ravel()


@pytest.fixture(scope="module")
def cfg5():
    from paper_1807_04180_b200.engine3 import DdmEngine3
    prob = config5()
    e = DdmEngine3(prob)
    yield prob, e
    e.close()


def test_config5_setup(cfg5):
    prob, e = cfg5
    ci = e.class_info()
    assert len(ci) == 8 and all(c["members"] == 1 for c in ci)   # mirror images
    assert all(c["factor_nnz"] == 83587619 for c in ci)
    assert all(c["probe_relres"] <= 1e-10 for c in ci)
    fp = e.footprint()
    assert 16 * 8 * fp["stored_values_per_class"] < 12e9            # 11.1 GB of factors
    assert fp["device_bytes_in_use"] < 40e9                         # front workspace released


def test_config5_apply_matches_numpy(cfg5):
    prob, e = cfg5
    rng = np.random.default_rng(11)
    u = rng.standard_normal(prob.n_global) + 1j * rng.standard_normal(prob.n_global)
    assert rel_l2(e.apply_global(u), _global_apply_numpy(prob, e.sigma0(), u)) <= 1e-13


def test_config5_fgmres_converges_and_is_linear(cfg5):
    from paper_1807_04180_b200.engine import DdmStats, FgmresOptions
    prob, e = cfg5
    f = prob.source_f()
    ps = DdmStats()
    x, res = e.fgmres(f, FgmresOptions(prob.tol, prob.max_iters, prob.restart), prob.k_steps, ps)
    assert res.converged and res.true_relres <= prob.tol
    # the true residual through an independent restatement of the operator
    r = f - _global_apply_numpy(prob, e.sigma0(), x)
    assert np.linalg.norm(r) / np.linalg.norm(f) <= prob.tol
    assert ps.solves == res.iters * prob.k_steps * prob.nsub  # every subdomain active
    z = e.precondition(f, 2)
    assert np.array_equal(e.precondition(2.0 * f, 2), 2.0 * z)
    mx, ncorr = e.refine_stats()
    assert mx <= 1e-11


def test_config5_local_solves(cfg5):
    prob, e = cfg5
    nw = int(np.prod(prob.window))
    rng = np.random.default_rng(5)
    b = rng.standard_normal(nw) + 1j * rng.standard_normal(nw)
    for c in (0, 7):
        x, rel = e.class_solve(c, b)
        assert rel <= 1e-11 and np.isfinite(x).all()


def test_config5_sweeps_match_restatement_fingerprint(cfg5):
    """precondition(f, K = 1, 2) at full size against the 3-D restatement's own run
    (tests/golden/make_golden_cfg5.py; its factorization took 35 min, so the vectors
    travel as 4096 seeded samples, 16 seeded projections and the norm)."""
    import os
    import sys
    from conftest import GOLDEN
    sys.path.insert(0, GOLDEN)
    from make_golden_cfg5 import fingerprint, fingerprint_basis
    prob, e = cfg5
    g = np.load(os.path.join(GOLDEN, "cfg5_fingerprint.npz"))
    idx, W = fingerprint_basis(prob.n_global)
    assert np.array_equal(idx, g["idx"])
    f = prob.source_f()
    for k in (1, 2):
        s, p, nrm = fingerprint(e.precondition(f, k), idx, W)
        assert rel_l2(s, g[f"z{k}_samples"]) <= 1e-10, k
        assert rel_l2(p, g[f"z{k}_proj"]) <= 1e-10, k
        assert abs(nrm - float(g[f"z{k}_norm"])) <= 1e-10 * float(g[f"z{k}_norm"]), k
