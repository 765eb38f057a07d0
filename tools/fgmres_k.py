"""FGMRES(30)+DDM(K) end to end (host b -> host x through the C-ABI) at small K,
where the per-iteration host round trip of a host-driven Arnoldi loop would show.

    python tools/fgmres_k.py [config] [K ...]       (HDDM_LIB selects the library)

Prints one JSON line per K: iterations, wall ms, ms per iteration, DDM it/s.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1807_04180_b200.engine import DdmEngine, FgmresOptions  # noqa: E402
from paper_1807_04180_b200.problems import config  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ks = [int(k) for k in sys.argv[2:]] or [1, 2]
    prob = config(cfg)
    b = prob.source_f()
    with DdmEngine(prob) as e:
        for K in ks:
            opt = FgmresOptions(prob.tol, prob.max_iters, prob.restart)
            e.fgmres(b, FgmresOptions(prob.tol, 2, prob.restart), K)  # warm-up (graphs, workspace)
            t0 = time.perf_counter()
            x, res = e.fgmres(b, opt, K)
            wall = time.perf_counter() - t0
            print(json.dumps({"lib": os.environ.get("HDDM_LIB", "libhddm.so"), "config": cfg,
                              "K": K, "iters": res.iters, "converged": res.converged,
                              "true_relres": res.true_relres, "wall_ms": 1e3 * wall,
                              "ms_per_iter": 1e3 * wall / max(res.iters, 1),
                              "ddm_it_per_s": res.iters * K / wall}), flush=True)


if __name__ == "__main__":
    main()
