"""The C restatement (oracle/hddm_oracle.c) pinned against the reference:
committed golden fixtures (always) and the live reference build (when
/root/reference was compiled into oracle/_ref). CPU only."""
import numpy as np
import pytest

import pyoracle
from conftest import golden, golden_cases, rel_l2

CASES = golden_cases()


@pytest.mark.parametrize("name,prob,run", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_golden(name, prob, run):
    g = golden(name)
    o = pyoracle.OracleEngine(prob)
    ci = o.class_info()
    assert [c["members"] for c in ci] == g["members"].tolist()
    assert [c["factor_nnz"] for c in ci] == g["factor_nnz"].tolist()
    assert np.allclose([c["probe_relres"] for c in ci], g["probe"], rtol=0, atol=1e-12)
    assert abs(o.sigma0 - float(g["sigma0"])) <= 1e-14 * float(g["sigma0"])
    f = prob.source_f()
    u, st = o.solve_iterative(f, 0.0, run["steps"])
    # bit-for-bit restatement (same operation order, -ffp-contract=off)
    assert rel_l2(u, g["u_steps"]) <= 1e-13
    assert (st.solves, st.skipped, st.steps) == (int(g["solves"]), int(g["skipped"]),
                                                 int(g["steps"]))
    assert np.allclose([h[1] for h in st.history], g["relres_hist"], rtol=1e-10, atol=0)
    if g["per_step"].size:
        for s in range(run["steps"]):
            z = o.precondition(f, s + 1)
            assert rel_l2(z, g["per_step"][s]) <= 1e-13
    if "apply_in" in g:
        assert rel_l2(o.apply_global(g["apply_in"]), g["apply_out"]) <= 1e-15
    if "fgmres" in run:
        fg = run["fgmres"]
        x, res, ps, zs = o.fgmres(f, fg["tol"], fg["max_iters"], fg["restart"], fg["K"], keep_z=3)
        assert res.iters == int(g["fg_iters"])
        assert rel_l2(x, g["fg_x"]) <= 1e-12
        assert np.allclose(res.history, g["fg_hist"], rtol=1e-8)
        assert (ps.solves, ps.skipped) == (int(g["fg_solves"]), int(g["fg_skipped"]))
        for k in range(len(zs)):
            assert rel_l2(zs[k], g["fg_z"][k]) <= 1e-12


needs_ref = pytest.mark.skipif(not pyoracle.ref_available(),
                               reason="reference not built here (oracle/_ref)")


@needs_ref
def test_oracle_bitwise_equal_to_live_reference():
    from paper_1807_04180_b200.problems import small
    prob = small(40, 2, 2, 4.0, 4, 8, source=("gaussian", 0.37, 0.58, 0.03))
    f = prob.source_f()
    o, r = pyoracle.OracleEngine(prob), pyoracle.RefEngine(prob)
    v = np.random.default_rng(5).standard_normal(prob.n_global) + 0j
    assert np.array_equal(o.apply_global(v), r.apply_global(v))
    uo, so = o.solve_iterative(f, 0.0, 5)
    ur, sr = r.solve_iterative(f, 0.0, 5)
    assert np.array_equal(uo, ur)
    assert (so.solves, so.skipped) == (sr.solves, sr.skipped)
    xo, ro, _, _ = o.fgmres(f, 1e-9, 30, 30, 1)
    xr, rr, _, _ = r.fgmres(f, 1e-9, 30, 30, 1)
    assert ro.iters == rr.iters and np.array_equal(xo, xr)


@needs_ref
def test_oracle_matches_reference_layered_thread_count():
    from paper_1807_04180_b200.problems import MEDIUM_LAYERED, random_layers, small
    lay = random_layers(4, seed=11)
    prob = small(48, 3, 2, 3.0, 4, 6, source=("point", 0.52, 0.47)).with_(
        medium_kind=MEDIUM_LAYERED, layers=lay)
    f = prob.source_f()
    o = pyoracle.OracleEngine(prob)
    for th in (1, 3):
        r = pyoracle.RefEngine(prob, threads=th)
        assert [c["members"] for c in o.class_info()] == [c["members"] for c in r.class_info()]
        uo, so = o.solve_iterative(f, 1e-10, 30)
        ur, sr = r.solve_iterative(f, 1e-10, 30)
        assert np.array_equal(uo, ur) and so.steps == sr.steps


def test_direct_solve_single_window_matches_one_sweep():
    """test_ddm.cpp:53-71: a 1x1 partition reproduces the direct solve in one
    sweep (the oracle's 1x1 engine IS a direct solve of the global window)."""
    from paper_1807_04180_b200.problems import small
    prob = small(40, 1, 1, 4.0, 4, 8, source=("point", 0.52, 0.47))
    o = pyoracle.OracleEngine(prob)
    u, st = o.solve_iterative(prob.source_f(), 1e-12, 5)
    assert st.converged and st.steps == 1 and st.solves == 1
    assert st.history[-1][1] <= 1e-12
