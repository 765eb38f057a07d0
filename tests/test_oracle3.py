"""The 3-D extension of the restatement (oracle/hddm_oracle3.c, BASELINE config 5).

The reference has no 3-D code, so this restatement cannot be pinned against it.
It is checked instead against (a) an independent numpy restatement of the 3-D
operator built from the same formulas (alpha_axis, the J-scaled 7-point stencil),
(b) a direct sparse solve of the global 3-D problem (the DDM-preconditioned
FGMRES must converge to it), and (c) structural properties (classes, ordering,
local-solve residuals, linearity). CPU only."""
import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import pyoracle
from conftest import rel_l2
from paper_1807_04180_b200.problems import Problem3, small3


def _alpha(m, c0, c1, lo, hi, prob, sigma0):
    h2, d = 0.5 * prob.h, prob.n_ramp * prob.h
    sig = 0.0

    def shifted(t, dsh):
        if t <= dsh:
            return 0.0
        if t >= dsh + d:
            return sigma0
        s = (t - dsh) / d
        return sigma0 * s * s
    if 2 * c0 - m > 0:
        sig += shifted((2 * c0 - m) * h2, prob.n_overlap * prob.h if lo else 0.0)
    if m - 2 * c1 > 0:
        sig += shifted((m - 2 * c1) * h2, prob.n_overlap * prob.h if hi else 0.0)
    return complex(1.0, sig)


def _global_matrix(prob: Problem3, sigma0: float):
    """L-form global operator (identity on the boundary shell), numpy/scipy."""
    dims = prob.gdims
    e = prob.n_ext
    ms = (prob.mx, prob.my, prob.mz)
    an, iah = [], []
    for a in range(3):
        n = dims[a]
        an.append(np.array([_alpha(2 * l, e, e + ms[a], 0, 0, prob, sigma0) for l in range(n)]))
        iah.append(np.array([1.0 / _alpha(2 * l + 1, e, e + ms[a], 0, 0, prob, sigma0)
                             for l in range(n)]))
    k2 = (prob.omega / prob.velocity) ** 2
    ih2 = 1.0 / (prob.h * prob.h)
    nx, ny, nz = dims
    rows, cols, vals = [], [], []
    idx = lambda p, q, r: (r * ny + q) * nx + p
    for r in range(nz):
        for q in range(ny):
            for p in range(nx):
                i = idx(p, q, r)
                if p in (0, nx - 1) or q in (0, ny - 1) or r in (0, nz - 1):
                    rows.append(i); cols.append(i); vals.append(1.0)
                    continue
                jac = an[0][p] * an[1][q] * an[2][r]
                ex, ey, ez = an[1][q] * an[2][r] * ih2, an[0][p] * an[2][r] * ih2, an[0][p] * an[1][q] * ih2
                terms = [(idx(p + 1, q, r), ex * iah[0][p]), (idx(p - 1, q, r), ex * iah[0][p - 1]),
                         (idx(p, q + 1, r), ey * iah[1][q]), (idx(p, q - 1, r), ey * iah[1][q - 1]),
                         (idx(p, q, r + 1), ez * iah[2][r]), (idx(p, q, r - 1), ez * iah[2][r - 1])]
                for j, c in terms:
                    rows.append(i); cols.append(j); vals.append(c / jac)
                rows.append(i); cols.append(i); vals.append(k2 - sum(c for _, c in terms) / jac)
    n = nx * ny * nz
    return sp.csr_matrix((np.array(vals, np.complex128), (rows, cols)), shape=(n, n))


@pytest.fixture(scope="module")
def prob():
    return small3(m=16, n=2, freq=3.0, n_ov=2, n_ramp=3)


@pytest.fixture(scope="module")
def ora(prob):
    return pyoracle.Oracle3Engine(prob)


def test_nd_order3_is_permutation_shell_first():
    nx, ny, nz = 11, 9, 13
    o = pyoracle.nd_order3(nx, ny, nz)
    assert sorted(o.tolist()) == list(range(nx * ny * nz))
    nshell = nx * ny * nz - (nx - 2) * (ny - 2) * (nz - 2)
    p, q, r = o % nx, (o // nx) % ny, o // (nx * ny)
    shell = (p == 0) | (q == 0) | (r == 0) | (p == nx - 1) | (q == ny - 1) | (r == nz - 1)
    assert shell[:nshell].all() and not shell[nshell:].any()
    # the last plane eliminated is the root separator: x = 1 + 9 // 2 (longest axis is z: 11)
    assert (r[-(nx - 2) * (ny - 2):] == 1 + 11 // 2).all()


def test_directions3():
    dirs = [pyoracle.direction3(d) for d in range(26)]
    assert len(set(dirs)) == 26 and (0, 0, 0) not in dirs
    lags = [sum(1 for v in d if v) for d in dirs]
    assert lags == [1] * 6 + [2] * 12 + [3] * 8


def test_apply_global_matches_numpy_restatement(prob, ora):
    A = _global_matrix(prob, ora.sigma0)
    rng = np.random.default_rng(3)
    u = rng.standard_normal(prob.n_global) + 1j * rng.standard_normal(prob.n_global)
    assert rel_l2(ora.apply_global(u), A @ u) <= 1e-13


def test_classes_and_local_solves(prob, ora):
    ci = ora.class_info()
    assert len(ci) == 8 and all(c["members"] == 1 for c in ci)  # mirror images
    assert len({c["factor_nnz"] for c in ci}) == 1
    assert all(c["probe_relres"] <= 1e-12 for c in ci)
    nw = int(np.prod(ora.window))
    rng = np.random.default_rng(1)
    b = rng.standard_normal(nw) + 1j * rng.standard_normal(nw)
    x, rel = ora.class_solve(3, b)
    r = b - ora.class_matvec(3, x)
    assert rel <= 1e-11 and np.linalg.norm(r) / np.linalg.norm(b) <= 1e-11
    # the assembled matrix is symmetric bit for bit (J-scaled stencil)
    for j in rng.integers(0, nw, 5):
        ej = np.zeros(nw, np.complex128); ej[j] = 1
        col = ora.class_matvec(3, ej)
        for i in np.nonzero(col)[0]:
            ei = np.zeros(nw, np.complex128); ei[i] = 1
            assert ora.class_matvec(3, ei)[j] == col[i]


def test_member_classes_4x4x4():
    p = small3(m=24, n=4, freq=2.0, n_ov=2, n_ramp=2)
    o = pyoracle.Oracle3Engine(p)
    mem = sorted(c["members"] for c in o.class_info())
    # per axis: low-boundary, interior (2 subdomains), high-boundary -> 3^3 classes
    assert len(mem) == 27
    assert sorted(mem) == sorted(a * b * c for a in (1, 2, 1) for b in (1, 2, 1) for c in (1, 2, 1))


def test_fgmres_converges_to_direct_solution(prob, ora):
    f = prob.source_f()
    x, res, ps, _ = ora.fgmres(f, 1e-10, 60, 30, prob.k_steps)
    assert res.converged and res.true_relres <= 1e-9
    A = _global_matrix(prob, ora.sigma0)
    xd = spla.spsolve(A.tocsc(), f)
    assert rel_l2(x, xd) <= 1e-7
    assert ps.solves > 0


def test_ddm_linearity_and_zero(prob, ora):
    f = prob.source_f()
    z1 = ora.precondition(f, 3)
    z2 = ora.precondition(2.0 * f, 3)
    assert np.array_equal(z2, 2.0 * z1)
    z0 = ora.precondition(np.zeros_like(f), 3)
    assert not z0.any()


def test_ddm_converges_standalone(prob, ora):
    u, st = ora.solve_iterative(prob.source_f(), 0.0, 6)
    rel = [h[1] for h in st.history]
    assert st.steps == 6 and st.solves == 48
    assert all(b < a for a, b in zip(rel, rel[1:]))
