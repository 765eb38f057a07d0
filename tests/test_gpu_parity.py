"""CUDA engine vs the reference (golden fixtures) and the C restatement on
identical inputs, through the C-ABI. Tolerances (BASELINE.json north_star):
per-iteration iterate rel-L2 <= 1e-10, final solution <= 1e-8, identical
iteration / solve / skip counts."""
import numpy as np
import pytest

import pyoracle
from conftest import golden, golden_cases, rel_l2

pytestmark = pytest.mark.gpu
CASES = golden_cases()
ITER_TOL = 1e-10
FINAL_TOL = 1e-8


@pytest.fixture(scope="module")
def engines():
    from paper_1807_04180_b200.engine import DdmEngine
    cache = {}

    def get(prob):
        if prob.name not in cache:
            cache[prob.name] = DdmEngine(prob)
        return cache[prob.name]
    yield get
    for e in cache.values():
        e.close()


@pytest.mark.parametrize("name,prob,run", CASES, ids=[c[0] for c in CASES])
def test_setup_matches_reference(engines, name, prob, run):
    g = golden(name)
    e = engines(prob)
    ci = e.class_info()
    assert [c["members"] for c in ci] == g["members"].tolist()
    assert [c["factor_nnz"] for c in ci] == g["factor_nnz"].tolist()
    assert all(c["backend"] == "ldlt" and c["probe_relres"] <= 1e-10 for c in ci)
    assert abs(e.sigma0() - float(g["sigma0"])) <= 1e-14 * float(g["sigma0"])


@pytest.mark.parametrize("name,prob,run", CASES, ids=[c[0] for c in CASES])
def test_standalone_iterates_match_reference(engines, name, prob, run):
    from paper_1807_04180_b200.engine import DdmStats
    g = golden(name)
    e = engines(prob)
    f = prob.source_f()
    st = DdmStats()
    u = e.solve_iterative(f, 0.0, run["steps"], st)
    assert rel_l2(u, g["u_steps"]) <= ITER_TOL
    assert (st.steps, st.solves, st.skipped) == (int(g["steps"]), int(g["solves"]),
                                                 int(g["skipped"]))
    assert [h.step for h in st.history] == list(range(1, run["steps"] + 1))
    np.testing.assert_allclose([h.relres for h in st.history], g["relres_hist"], rtol=1e-6, atol=1e-10)
    if g["per_step"].size:
        for s in range(run["steps"]):
            z = e.precondition(f, s + 1)
            assert rel_l2(z, g["per_step"][s]) <= ITER_TOL, s


@pytest.mark.parametrize("name,prob,run", [c for c in CASES if "fgmres" in c[2]],
                         ids=[c[0] for c in CASES if "fgmres" in c[2]])
def test_fgmres_matches_reference(engines, name, prob, run):
    from paper_1807_04180_b200.engine import DdmStats, FgmresOptions
    g = golden(name)
    e = engines(prob)
    fg = run["fgmres"]
    ps = DdmStats()
    x, res = e.fgmres(prob.source_f(), FgmresOptions(fg["tol"], fg["max_iters"], fg["restart"]),
                      fg["K"], ps)
    assert res.iters == int(g["fg_iters"]) and res.converged
    assert rel_l2(x, g["fg_x"]) <= FINAL_TOL
    np.testing.assert_allclose(res.history, g["fg_hist"], rtol=1e-6, atol=1e-10)
    assert (ps.solves, ps.skipped) == (int(g["fg_solves"]), int(g["fg_skipped"]))
    assert abs(res.true_relres - float(g["fg_true"])) <= 1e-6 * float(g["fg_true"]) + 1e-10


@pytest.mark.parametrize("name,prob,run", CASES[:2], ids=[c[0] for c in CASES[:2]])
def test_apply_global_matches_reference(engines, name, prob, run):
    g = golden(name)
    e = engines(prob)
    assert rel_l2(e.apply_global(g["apply_in"]), g["apply_out"]) <= 1e-14


def test_local_class_solves_match_oracle(engines):
    """Batched supernodal solve vs the restatement's Factorization::solve."""
    from paper_1807_04180_b200.problems import config
    prob = config(1)
    e = engines(prob)
    o = pyoracle.OracleEngine(prob)
    nx, ny = e.window_dims()
    rng = np.random.default_rng(11)
    for c in range(len(e.class_info())):
        b = rng.standard_normal(nx * ny) + 1j * rng.standard_normal(nx * ny)
        xg, rg = e.class_solve(c, b)
        xo, ro = o.class_solve(c, b)
        assert rel_l2(xg, xo) <= 1e-12
        assert rg <= 1e-11


def test_subdomain_taps_match_oracle(engines):
    """Per-subdomain right-hand sides (gather-sources kernels) and local
    solutions after a step, against the restatement."""
    from paper_1807_04180_b200.problems import small
    prob = small(80, 2, 2, 8.0, 10, 20, source=("gaussian", 0.41, 0.63, 0.02))
    e = engines(prob)
    o = pyoracle.OracleEngine(prob)
    f = prob.source_f()
    for K in (1, 2, 3):
        e.precondition(f, K)
        o.precondition(f, K)
        taps = [(e.tap_subdomain(t), o.tap_subdomain(t)) for t in range(prob.nsub)]
        # subdomains whose incoming sources are still rounding-level (cancellation
        # in L_t(beta v) where the taper is flat) are compared on the scale of
        # the largest local solution of the step
        scale_r = max(np.linalg.norm(ro) for (_, (ro, _, _)) in taps)
        scale_u = max(np.linalg.norm(uo) for (_, (_, uo, _)) in taps)
        for (rg, ug, ag), (ro, uo, ao) in taps:
            assert ag == ao
            if ag:
                assert np.linalg.norm(rg - ro) <= 1e-7 * scale_r
                assert np.linalg.norm(ug - uo) <= ITER_TOL * scale_u


def test_lens_medium_matches_oracle():
    """BASELINE config 3's medium kind (reference extension), small grid."""
    from paper_1807_04180_b200.engine import DdmEngine, DdmStats
    from paper_1807_04180_b200.problems import MEDIUM_LENS, small
    prob = small(64, 4, 4, 6.0, 4, 8, source=("gaussian", 0.25, 0.25, 0.02)).with_(
        medium_kind=MEDIUM_LENS, lens=(0.4, 0.5, 0.5, 0.05))
    e = DdmEngine(prob)
    o = pyoracle.OracleEngine(prob)
    assert [c["members"] for c in e.class_info()] == [c["members"] for c in o.class_info()]
    f = prob.source_f()
    st = DdmStats()
    u = e.solve_iterative(f, 0.0, 6, st)
    uo, so = o.solve_iterative(f, 0.0, 6)
    assert rel_l2(u, uo) <= ITER_TOL and (st.solves, st.skipped) == (so.solves, so.skipped)
    e.close()


@pytest.mark.parametrize("cfg", [2, 3])
def test_fullsize_fgmres_matches_oracle(cfg):
    """BASELINE configs 2 and 3 end to end at full size (1024^2, 8x8,
    FGMRES(30)+DDM(K=16); config 3 is the lens medium, 64 distinct windows)
    against the C restatement (pinned bit-for-bit to the reference by
    test_oracle; for the lens medium, which the reference lacks, the same
    formulas with the clamped lens k^2): identical iteration count and solve /
    skip counts, final x <= 1e-8, the first preconditioner application <= 1e-10."""
    from paper_1807_04180_b200.engine import DdmEngine, DdmStats, FgmresOptions
    from paper_1807_04180_b200.problems import config
    prob = config(cfg)
    e = DdmEngine(prob)
    o = pyoracle.OracleEngine(prob)
    f = prob.source_f()
    ps = DdmStats()
    x, res = e.fgmres(f, FgmresOptions(prob.tol, prob.max_iters, prob.restart), prob.k_steps, ps)
    xo, ro, pso, zo = o.fgmres(f, prob.tol, prob.max_iters, prob.restart, prob.k_steps, keep_z=1)
    assert res.iters == ro.iters and res.converged == ro.converged
    assert rel_l2(x, xo) <= FINAL_TOL
    assert (ps.solves, ps.skipped) == (pso.solves, pso.skipped)
    z = e.precondition(f / np.linalg.norm(f), prob.k_steps)
    assert rel_l2(z, zo[0]) <= ITER_TOL
    e.close()


@pytest.mark.parametrize("n1,n2", [(1, 1), (3, 1), (1, 3), (3, 2), (5, 4)])
def test_partition_shapes_match_oracle(n1, n2):
    """Single-subdomain and non-square partitions (a single window: no
    transfers; 1-3 member classes; mixed tile groups), layered medium so x and y
    differ: per-step iterates and residual history, solve/skip counts, the
    preconditioner on several random inputs, and FGMRES up to its first
    stagnating iteration (at a near-breakdown the Arnoldi normalisation cancels
    and last-bit differences in the reduction order steer both codes apart --
    the reference's own result depends on its summation order there)."""
    from paper_1807_04180_b200.engine import DdmEngine, DdmStats, FgmresOptions
    from paper_1807_04180_b200.problems import MEDIUM_LAYERED, small
    prob = small(24 * n1, n1, n2, 3.0, 3, 6, source=("gaussian", 0.4, 0.55, 0.05)).with_(
        my=24 * n2, medium_kind=MEDIUM_LAYERED,
        layers=[(0.0, 0.3, 1.0), (0.3, 0.7, 1.6), (0.7, 1.0, 1.2)])
    e = DdmEngine(prob)
    o = pyoracle.OracleEngine(prob)
    assert [c["members"] for c in e.class_info()] == [c["members"] for c in o.class_info()]
    f = prob.source_f()
    st = DdmStats()
    u = e.solve_iterative(f, 0.0, 5, st)
    uo, so = o.solve_iterative(f, 0.0, 5)
    assert rel_l2(u, uo) <= ITER_TOL
    assert (st.steps, st.solves, st.skipped) == (so.steps, so.solves, so.skipped)
    for a, b in zip(st.history, so.history):
        assert abs(a.relres - b[1]) <= 1e-10 * abs(b[1]) + 1e-13
    rng = np.random.default_rng(n1 * 10 + n2)
    K = n1 + n2
    for _ in range(3):  # repeated applications: no state carried between calls
        r = interior_noise(prob, rng)
        sa, sb = DdmStats(), pyoracle.Stats()
        assert rel_l2(e.precondition(r, K, sa), o.precondition(r, K, sb)) <= ITER_TOL
        assert (sa.solves, sa.skipped) == (sb.solves, sb.skipped)
    x, res = e.fgmres(f, FgmresOptions(1e-8, 30, 30), K)
    xo, ro, _, _ = o.fgmres(f, 1e-8, 30, 30, K, keep_z=0)
    prev = None
    for a, b in zip(res.history, ro.history):
        if prev is not None and b >= 0.999 * prev:
            break  # stagnation: beyond here the comparison is not meaningful
        assert abs(a - b) <= 1e-8 * abs(b) + 1e-13
        prev = b
    if ro.converged and all(ro.history[k] < 0.999 * ro.history[k - 1] for k in range(1, ro.iters)):
        assert res.iters == ro.iters and rel_l2(x, xo) <= FINAL_TOL
    e.close()


def interior_noise(prob, rng):
    r = rng.standard_normal(prob.n_global) + 1j * rng.standard_normal(prob.n_global)
    r = r.reshape(prob.gny, prob.gnx)
    r[0, :] = r[-1, :] = r[:, 0] = r[:, -1] = 0
    return r.ravel()
