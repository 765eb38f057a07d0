"""Fingerprints of BASELINE config 5 (3-D) from the 3-D restatement at full size.

The restatement's single-threaded factorization of the eight 57^3 windows takes ~35 min
(measured here: 2124 s; then 5.9 s for the first sweep and 3.7 s per later sweep), too
long for a test, so its outputs travel as fingerprints: precondition(f, K) for K = 1, 2
sampled at 4096 seeded positions, 16 projections on seeded complex Gaussian vectors, and
the norm. tests/test_gpu_3d.py compares the GPU engine's vectors with them.

    python tests/golden/make_golden_cfg5.py [z1.npy z2.npy]   (precomputed vectors optional)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def fingerprint_basis(n: int):
    rng = np.random.default_rng(20261020)
    idx = np.sort(rng.choice(n, 4096, replace=False))
    W = rng.standard_normal((16, n)) + 1j * rng.standard_normal((16, n))
    return idx, W


def fingerprint(z, idx, W):
    return z[idx], W.conj() @ z, np.linalg.norm(z)


def main():
    from paper_1807_04180_b200.problems import config5
    prob = config5()
    f = prob.source_f()
    if len(sys.argv) == 3:
        zs = [np.load(sys.argv[1]), np.load(sys.argv[2])]
    else:
        import pyoracle
        o = pyoracle.Oracle3Engine(prob)
        zs = [o.precondition(f, 1), o.precondition(f, 2)]
    idx, W = fingerprint_basis(prob.n_global)
    out = {"idx": idx}
    for k, z in enumerate(zs, 1):
        s, p, nrm = fingerprint(z, idx, W)
        out[f"z{k}_samples"], out[f"z{k}_proj"], out[f"z{k}_norm"] = s, p, nrm
    np.savez_compressed(os.path.join(HERE, "cfg5_fingerprint.npz"), **out)


if __name__ == "__main__":
    main()
