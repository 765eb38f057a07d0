"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (needs /root/reference compiled by `make -C oracle ref`):
    python tests/golden/make_golden.py
It writes tests/golden/*.npz. The GPU box has no /root/reference; the tests
there compare against these files and against the C restatement (oracle/),
whose parity with the reference these same fixtures pin.

Cases (seeded synthetic inputs; no external data):
  small_point   : reference test make_cfg(40, 2, 2, 4.0, 4, 8), point source
                  (proj/tests/test_ddm.cpp:15-30), 6 standalone steps
  small_gauss   : make_cfg(80, 2, 2, 8.0, 10, 20), Gaussian source, 5 steps
                  and FGMRES(30)+DDM(K=2)
  cfg1          : BASELINE config 1 (256^2, 4x4, ov 4, PML 16, w=40pi) --
                  10 standalone steps: final field + per-step relres
  layered_small : 96^2, 4x4, ov 4, PML 8, 5 random layers (mt19937_64 seed 3),
                  FGMRES(30)+DDM(K=8) to 1e-8
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_1807_04180_b200.problems import config, small, random_layers, MEDIUM_LAYERED  # noqa
import pyoracle  # noqa


def cases():
    yield "small_point", small(40, 2, 2, 4.0, 4, 8, source=("point", 0.3, 0.6)), dict(steps=6)
    yield "small_gauss", small(80, 2, 2, 8.0, 10, 20, source=("gaussian", 0.41, 0.63, 0.02)), \
        dict(steps=5, fgmres=dict(tol=1e-8, max_iters=40, restart=30, K=2))
    yield "cfg1", config(1), dict(steps=10)
    lay = random_layers(5, seed=3)
    cmin = min(c for *_, c in lay)
    p = small(96, 4, 4, 1.0, 4, 8, source=("gaussian", 0.5, 0.2, 0.02))
    p = p.with_(name="layered_small", medium_kind=MEDIUM_LAYERED, layers=lay,
                omega=2 * np.pi * cmin * 96 / 10)
    yield "layered_small", p, dict(steps=4, fgmres=dict(tol=1e-8, max_iters=60, restart=30, K=8))


def main():
    for name, prob, run in cases():
        ref = pyoracle.RefEngine(prob, threads=1)
        f = prob.source_f()
        out = {"f_norm": np.linalg.norm(f)}
        u, st = ref.solve_iterative(f, 0.0, run["steps"])
        out.update(u_steps=u, relres_hist=np.array([h[1] for h in st.history]),
                   solves=st.solves, skipped=st.skipped, steps=st.steps)
        # per-step iterates via precondition(f, K=s) (ddm.cpp:280-287)
        per = [ref.precondition(f, s) for s in range(1, run["steps"] + 1)]
        small_case = prob.n_global * run["steps"] < 500_000
        out["per_step"] = np.array(per) if small_case else np.zeros(0)
        ci = ref.class_info()
        out["members"] = np.array([c["members"] for c in ci])
        out["factor_nnz"] = np.array([c["factor_nnz"] for c in ci])
        out["probe"] = np.array([c["probe_relres"] for c in ci])
        out["sigma0"] = ref.sigma0
        if small_case:
            rng = np.random.default_rng(7)
            v = rng.standard_normal(prob.n_global) + 1j * rng.standard_normal(prob.n_global)
            out["apply_in"] = v
            out["apply_out"] = ref.apply_global(v)
        if "fgmres" in run:
            fg = run["fgmres"]
            x, res, ps, zs = ref.fgmres(f, fg["tol"], fg["max_iters"], fg["restart"], fg["K"],
                                        keep_z=3)
            out.update(fg_x=x, fg_iters=res.iters, fg_hist=np.array(res.history),
                       fg_true=res.true_relres, fg_z=zs, fg_solves=ps.solves,
                       fg_skipped=ps.skipped)
        ref.close()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
