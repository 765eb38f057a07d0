"""Host-side flexible GMRES over caller-supplied operators: the reference's
`fgmres(n, A, M, b, x, opt)` with `LinearOp` callbacks (proj/include/helmddm/
krylov.hpp:31-33, krylov.cpp:24-133), restated.

The production path is the device-resident `DdmEngine.fgmres` (A = apply_global,
M = precondition, wired as cli.cpp:210-228). This generic form keeps the
reference API for host-lambda use -- e.g. the reference's own FGMRES driving the
GPU preconditioner, which isolates preconditioner parity.

Algorithm (the reference's): right-preconditioned FGMRES from x = 0, modified
Gram-Schmidt Arnoldi, complex Givens rotations on the Hessenberg columns, the
recursive residual |g_{j+1}| / |b| per iteration, cyclic restart with the
residual recomputed explicitly, stop on tol, on a dead column (zero rotation
norm) or an invariant subspace (zero new basis norm); the true residual of the
returned x at the end.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

LinearOp = Callable[[np.ndarray], np.ndarray]


@dataclass
class FgmresOptions:
    """helmddm::FgmresOptions (krylov.hpp:11-15)."""
    tol: float = 1e-6
    max_iters: int = 200
    restart: int = 0  # 0: no restart


@dataclass
class FgmresResult:
    """helmddm::FgmresResult (krylov.hpp:17-25)."""
    iters: int = 0
    converged: bool = False
    relres: float = -1.0
    true_relres: float = -1.0
    history: List[float] = field(default_factory=list)
    iter_ms: List[float] = field(default_factory=list)


def fgmres(n: int, A: LinearOp, M: Optional[LinearOp], b: np.ndarray,
           opt: FgmresOptions) -> tuple:
    """Returns (x, FgmresResult). A(v) and M(v) map complex128 length-n arrays to
    new arrays; M None means no preconditioner (Z_j = V_j)."""
    b = np.ascontiguousarray(b, np.complex128)
    if b.shape != (n,):
        raise ValueError("b must have n entries")
    res = FgmresResult()
    x = np.zeros(n, np.complex128)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        res.converged = True
        res.relres = res.true_relres = 0.0
        return x, res
    r = b.copy()
    total = 0
    stop = False
    while not stop and total < opt.max_iters:
        m = min(opt.restart, opt.max_iters - total) if opt.restart > 0 else opt.max_iters - total
        rnorm = float(np.linalg.norm(r))
        if rnorm == 0.0:
            res.converged = True
            break
        V = [r / rnorm]
        Z: List[np.ndarray] = []
        H = np.zeros((m + 1, m), np.complex128)  # H[i, j]: row i of column j
        g = np.zeros(m + 1, np.complex128)
        g[0] = rnorm
        cs = np.zeros(m)
        sn = np.zeros(m, np.complex128)
        k = 0
        for j in range(m):
            t0 = time.perf_counter()
            z = np.asarray(M(V[j]) if M is not None else V[j], np.complex128)
            Z.append(z)
            w = np.array(A(z), dtype=np.complex128)
            for i in range(j + 1):  # modified Gram-Schmidt
                hij = np.vdot(V[i], w)
                H[i, j] = hij
                w -= hij * V[i]
            hlast = float(np.linalg.norm(w))
            H[j + 1, j] = hlast
            for i in range(j):  # previous rotations on the new column
                a, c = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * a + sn[i] * c
                H[i + 1, j] = -np.conj(sn[i]) * a + cs[i] * c
            a, c = H[j, j], H[j + 1, j]
            tnorm = float(np.sqrt(abs(a) ** 2 + abs(c) ** 2))
            if tnorm == 0.0:  # dead column: dropped, stop
                stop = True
                break
            if a == 0:
                cs[j] = 0.0
                sn[j] = np.conj(c) / abs(c)
            else:
                cs[j] = abs(a) / tnorm
                sn[j] = (a / abs(a)) * np.conj(c) / tnorm
            H[j, j] = cs[j] * a + sn[j] * c
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            k = j + 1
            res.relres = float(abs(g[j + 1])) / bnorm
            res.history.append(res.relres)
            res.iter_ms.append((time.perf_counter() - t0) * 1e3)
            if res.relres <= opt.tol:
                res.converged = True
                stop = True
                break
            if hlast == 0.0:  # invariant subspace
                stop = True
                break
            V.append(w / hlast)
        if k > 0:  # back substitution on the rotated triangle, x += Z y
            y = np.zeros(k, np.complex128)
            for i in range(k - 1, -1, -1):
                y[i] = (g[i] - np.dot(H[i, i + 1:k], y[i + 1:k])) / H[i, i]
            for l in range(k):
                x += y[l] * Z[l]
        if not stop:  # restart from the explicit residual
            r = b - np.asarray(A(x), np.complex128)
    res.iters = total
    res.true_relres = float(np.linalg.norm(b - np.asarray(A(x), np.complex128))) / bnorm
    return x, res
