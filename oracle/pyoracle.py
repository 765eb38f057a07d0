"""ctypes front end for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``OracleEngine`` -- the C restatement ``oracle/hddm_oracle.c`` (kind "port").
* ``RefEngine``    -- the UNMODIFIED reference sources compiled by
  ``oracle/Makefile`` into ``oracle/_ref/libhelmddm_ref.so`` (kind "reference").

Both expose the same Python surface, mirroring ``DdmEngine``
(proj/include/helmddm/ddm.hpp:53-109) and ``fgmres`` (krylov.hpp:31-33), so a
test can run either side on identical inputs. Only tests/, __graft_entry__.smoke()
and bench.py's reference / cpu_baseline legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
ORACLE_SO = os.path.join(REF_DIR, "liboracle.so")
REF_SO = os.path.join(REF_DIR, "libhelmddm_ref.so")


class _Problem(C.Structure):
    _fields_ = [
        ("x0", C.c_double), ("y0", C.c_double), ("h", C.c_double),
        ("mx", C.c_int), ("my", C.c_int), ("n1", C.c_int), ("n2", C.c_int),
        ("n_overlap", C.c_int), ("n_ramp", C.c_int),
        ("omega", C.c_double), ("medium_kind", C.c_int), ("velocity", C.c_double),
        ("n_layers", C.c_int),
        ("layer_ylo", C.POINTER(C.c_double)), ("layer_yhi", C.POINTER(C.c_double)),
        ("layer_c", C.POINTER(C.c_double)),
        ("c_sigma", C.c_double), ("sigma0", C.c_double), ("threads", C.c_int),
        # oracle-only tail (lens); the reference struct stops before it
        ("lens_amp", C.c_double), ("lens_xc", C.c_double), ("lens_yc", C.c_double),
        ("lens_w", C.c_double),
    ]


class _Stats(C.Structure):
    _fields_ = [("steps", C.c_int), ("solves", C.c_long), ("skipped", C.c_long),
                ("relres", C.c_double), ("converged", C.c_int),
                ("factor_ms", C.c_double), ("sweep_ms", C.c_double)]


class _FgOut(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("relres", C.c_double),
                ("true_relres", C.c_double), ("wall_ms", C.c_double)]


@dataclass
class Stats:
    steps: int = 0
    solves: int = 0
    skipped: int = 0
    relres: float = -1.0
    converged: bool = False
    factor_ms: float = 0.0
    sweep_ms: float = 0.0
    history: Optional[list] = None


@dataclass
class FgmresResult:
    iters: int
    converged: bool
    relres: float
    true_relres: float
    history: List[float]
    wall_ms: float


def build(ref: bool = False) -> None:
    """Build the restatement (and, if asked and /root/reference exists, the
    reference) with oracle/Makefile."""
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _load(path: str, prefix: str):
    if not os.path.exists(path):
        if prefix == "orc":
            build(False)
        else:
            raise FileNotFoundError(f"{path} missing (build with `make -C oracle ref`)")
    lib = C.CDLL(path)
    P = C.POINTER
    d = C.c_double
    dp = P(C.c_double)
    vp = C.c_void_p
    ip = P(C.c_int)
    sig = {
        "last_error": (C.c_char_p, []),
        "create": (C.c_int, [P(_Problem), P(vp)]),
        "destroy": (None, [vp]),
        "n_global": (C.c_long, [vp]),
        "sigma0": (d, [vp]),
        "num_classes": (C.c_int, [vp]),
        "class_info": (C.c_int, [vp, C.c_int, ip, P(C.c_long), dp, ip]),
        "apply_global": (C.c_int, [vp, dp, dp]),
        "solve_iterative": (C.c_int, [vp, dp, d, C.c_int, C.c_int, dp, P(_Stats), ip, dp,
                                      C.c_int, ip]),
        "precondition": (C.c_int, [vp, dp, dp, C.c_int, P(_Stats)]),
        "fgmres": (C.c_int, [vp, dp, dp, d, C.c_int, C.c_int, C.c_int, P(_FgOut), dp,
                             C.c_int, dp, C.c_int, P(_Stats)]),
    }
    if prefix == "orc":
        sig.update({
            "tap_subdomain": (C.c_int, [vp, C.c_int, dp, dp, ip]),
            "class_solve": (C.c_int, [vp, C.c_int, dp, dp, dp]),
            "class_of": (C.c_int, [vp, C.c_int]),
            "window_dims": (C.c_int, [vp, ip, ip]),
            "nd_order": (C.c_int, [C.c_int, C.c_int, ip]),
        })
    else:
        sig["factor_ms"] = (d, [vp])
        sig["direct_solve"] = (C.c_int, [P(_Problem), dp, dp])
    for name, (res, args) in sig.items():
        fn = getattr(lib, f"{prefix}_{name}")
        fn.restype = res
        fn.argtypes = args
    return lib


_LIBS = {}


def _lib(kind: str):
    if kind not in _LIBS:
        _LIBS[kind] = _load(ORACLE_SO, "orc") if kind == "orc" else _load(REF_SO, "ref")
    return _LIBS[kind]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _cvec(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    return a


class _Engine:
    prefix = "orc"

    def __init__(self, prob, threads: int = 1):
        self.prob = prob
        self.lib = _lib(self.prefix)
        fn = lambda n: getattr(self.lib, f"{self.prefix}_{n}")
        self._fn = fn
        lay = prob.layers or [(0.0, 0.0, 1.0)]
        self._ylo = np.array([l[0] for l in lay], np.float64)
        self._yhi = np.array([l[1] for l in lay], np.float64)
        self._c = np.array([l[2] for l in lay], np.float64)
        P = _Problem()
        P.x0, P.y0, P.h = prob.x0, prob.y0, prob.h
        P.mx, P.my, P.n1, P.n2 = prob.mx, prob.my, prob.n1, prob.n2
        P.n_overlap, P.n_ramp = prob.n_overlap, prob.n_ramp
        P.omega, P.medium_kind, P.velocity = prob.omega, prob.medium_kind, prob.velocity
        P.n_layers = len(prob.layers)
        P.layer_ylo, P.layer_yhi, P.layer_c = _dp(self._ylo), _dp(self._yhi), _dp(self._c)
        P.c_sigma, P.sigma0, P.threads = prob.c_sigma, prob.sigma0, threads
        P.lens_amp, P.lens_xc, P.lens_yc, P.lens_w = prob.lens
        if self.prefix == "ref" and prob.medium_kind not in (0, 1):
            raise ValueError("the reference has no lens medium (SURVEY 8(c))")
        self._P = P
        h = C.c_void_p()
        rc = fn("create")(C.byref(P), C.byref(h))
        if rc != 0:
            raise RuntimeError(f"{self.prefix}_create failed ({rc}): "
                               f"{fn('last_error')().decode()}")
        self.h = h
        self.n = int(fn("n_global")(h))

    def close(self):
        if self.h:
            self._fn("destroy")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"{self.prefix} error {rc}: {self._fn('last_error')().decode()}")

    @property
    def sigma0(self) -> float:
        return float(self._fn("sigma0")(self.h))

    def class_info(self):
        out = []
        for c in range(self._fn("num_classes")(self.h)):
            m, nnz, pr, ld = C.c_int(), C.c_long(), C.c_double(), C.c_int()
            self._check(self._fn("class_info")(self.h, c, C.byref(m), C.byref(nnz),
                                               C.byref(pr), C.byref(ld)))
            out.append(dict(members=m.value, factor_nnz=nnz.value, probe_relres=pr.value,
                            backend="ldlt" if ld.value else "lu"))
        return out

    def apply_global(self, u) -> np.ndarray:
        u = _cvec(u)
        out = np.empty_like(u)
        self._check(self._fn("apply_global")(self.h, _dp(u), _dp(out)))
        return out

    def solve_iterative(self, f, tol: float, max_steps: int, check_every: int = 1):
        f = _cvec(f)
        out = np.empty_like(f)
        st = _Stats()
        cap = max_steps + 1
        hs = np.zeros(cap, np.int32)
        hr = np.zeros(cap, np.float64)
        hl = C.c_int()
        self._check(self._fn("solve_iterative")(
            self.h, _dp(f), tol, max_steps, check_every, _dp(out), C.byref(st),
            hs.ctypes.data_as(C.POINTER(C.c_int)), _dp(hr), cap, C.byref(hl)))
        s = Stats(st.steps, st.solves, st.skipped, st.relres, bool(st.converged),
                  st.factor_ms, st.sweep_ms,
                  [(int(hs[i]), float(hr[i])) for i in range(min(hl.value, cap))])
        return out, s

    def precondition(self, r, ksteps: int, stats: Optional[Stats] = None):
        r = _cvec(r)
        z = np.empty_like(r)
        st = _Stats()
        self._check(self._fn("precondition")(self.h, _dp(r), _dp(z), ksteps, C.byref(st)))
        if stats is not None:
            stats.solves += st.solves
            stats.skipped += st.skipped
            stats.sweep_ms += st.sweep_ms
        return z

    def fgmres(self, b, tol: float, max_iters: int, restart: int, K: int,
               keep_z: int = 0):
        b = _cvec(b)
        x = np.empty_like(b)
        res = _FgOut()
        hist = np.zeros(max(max_iters, 1), np.float64)
        zs = np.zeros((keep_z, self.n), np.complex128) if keep_z else None
        pst = _Stats()
        self._check(self._fn("fgmres")(
            self.h, _dp(b), _dp(x), tol, max_iters, restart, K, C.byref(res), _dp(hist),
            len(hist), _dp(zs) if keep_z else None, keep_z, C.byref(pst)))
        r = FgmresResult(res.iters, bool(res.converged), res.relres, res.true_relres,
                         list(hist[:res.iters]), res.wall_ms)
        ps = Stats(solves=pst.solves, skipped=pst.skipped, sweep_ms=pst.sweep_ms)
        return x, r, ps, (zs[:min(keep_z, res.iters)] if keep_z else None)


class OracleEngine(_Engine):
    """The C restatement (oracle/hddm_oracle.c)."""
    prefix = "orc"

    def tap_subdomain(self, t: int):
        nx, ny = C.c_int(), C.c_int()
        self._fn("window_dims")(self.h, C.byref(nx), C.byref(ny))
        nw = nx.value * ny.value
        rhs = np.zeros(nw, np.complex128)
        u = np.zeros(nw, np.complex128)
        act = C.c_int()
        self._check(self._fn("tap_subdomain")(self.h, t, _dp(rhs), _dp(u), C.byref(act)))
        return rhs, u, bool(act.value)

    def class_of(self, t: int) -> int:
        return int(self._fn("class_of")(self.h, t))

    def class_solve(self, c: int, b):
        b = _cvec(b)
        x = np.empty_like(b)
        rel = C.c_double()
        self._check(self._fn("class_solve")(self.h, c, _dp(b), _dp(x), C.byref(rel)))
        return x, rel.value


class RefEngine(_Engine):
    """The unmodified reference (oracle/_ref/libhelmddm_ref.so)."""
    prefix = "ref"

    @property
    def factor_ms(self) -> float:
        return float(self._fn("factor_ms")(self.h))


def nd_order(nx: int, ny: int) -> np.ndarray:
    out = np.zeros(nx * ny, np.int32)
    _lib("orc").orc_nd_order(nx, ny, out.ctypes.data_as(C.POINTER(C.c_int)))
    return out


def ref_direct_solve(prob, f) -> np.ndarray:
    eng = RefEngine.__new__(RefEngine)
    lib = _lib("ref")
    f = _cvec(f)
    out = np.empty_like(f)
    P = _Problem()
    P.x0, P.y0, P.h = prob.x0, prob.y0, prob.h
    P.mx, P.my, P.n1, P.n2 = prob.mx, prob.my, prob.n1, prob.n2
    P.n_overlap, P.n_ramp = prob.n_overlap, prob.n_ramp
    P.omega, P.medium_kind, P.velocity = prob.omega, prob.medium_kind, prob.velocity
    lay = prob.layers or [(0.0, 0.0, 1.0)]
    ylo = np.array([l[0] for l in lay]); yhi = np.array([l[1] for l in lay])
    cc = np.array([l[2] for l in lay])
    P.n_layers = len(prob.layers)
    P.layer_ylo, P.layer_yhi, P.layer_c = _dp(ylo), _dp(yhi), _dp(cc)
    P.c_sigma, P.sigma0, P.threads = prob.c_sigma, prob.sigma0, 1
    rc = lib.ref_direct_solve(C.byref(P), _dp(f), _dp(out))
    if rc:
        raise RuntimeError(lib.ref_last_error().decode())
    del eng
    return out


# ------------------------------------------------------------------ 3-D
class _Problem3(C.Structure):
    _fields_ = [
        ("x0", C.c_double), ("y0", C.c_double), ("z0", C.c_double), ("h", C.c_double),
        ("mx", C.c_int), ("my", C.c_int), ("mz", C.c_int),
        ("n1", C.c_int), ("n2", C.c_int), ("n3", C.c_int),
        ("n_overlap", C.c_int), ("n_ramp", C.c_int),
        ("omega", C.c_double), ("velocity", C.c_double),
        ("c_sigma", C.c_double), ("sigma0", C.c_double),
    ]


def _lib3():
    lib = _lib("orc")
    if getattr(lib, "_have3", False):
        return lib
    P = C.POINTER
    d = C.c_double
    dp = P(C.c_double)
    vp = C.c_void_p
    ip = P(C.c_int)
    sig = {
        "create": (C.c_int, [P(_Problem3), P(vp)]),
        "destroy": (None, [vp]),
        "n_global": (C.c_long, [vp]),
        "sigma0": (d, [vp]),
        "num_classes": (C.c_int, [vp]),
        "class_of": (C.c_int, [vp, C.c_int]),
        "window_dims": (C.c_int, [vp, ip]),
        "class_info": (C.c_int, [vp, C.c_int, ip, P(C.c_long), dp]),
        "class_solve": (C.c_int, [vp, C.c_int, dp, dp, dp]),
        "class_matvec": (C.c_int, [vp, C.c_int, dp, dp]),
        "apply_global": (C.c_int, [vp, dp, dp]),
        "solve_iterative": (C.c_int, [vp, dp, d, C.c_int, C.c_int, dp, P(_Stats), ip, dp,
                                      C.c_int, ip]),
        "precondition": (C.c_int, [vp, dp, dp, C.c_int, P(_Stats)]),
        "fgmres": (C.c_int, [vp, dp, dp, d, C.c_int, C.c_int, C.c_int, P(_FgOut), dp,
                             C.c_int, dp, C.c_int, P(_Stats)]),
        "tap_subdomain": (C.c_int, [vp, C.c_int, dp, dp, ip]),
        "nd_order": (C.c_int, [C.c_int, C.c_int, C.c_int, ip]),
        "direction": (C.c_int, [C.c_int, ip]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, f"orc3_{name}")
        fn.restype = res
        fn.argtypes = args
    lib._have3 = True
    return lib


class Oracle3Engine(_Engine):
    """The 3-D extension of the restatement (oracle/hddm_oracle3.c). Parity
    unpinned: the reference has no 3-D code."""
    prefix = "orc3"

    def __init__(self, prob):  # noqa: D401 -- same surface as _Engine
        self.prob = prob
        self.lib = _lib3()
        fn = lambda n: getattr(self.lib, f"orc3_{n}") if n != "last_error" else self.lib.orc_last_error
        self._fn = fn
        P = _Problem3()
        P.x0, P.y0, P.z0, P.h = prob.x0, prob.y0, prob.z0, prob.h
        P.mx, P.my, P.mz = prob.mx, prob.my, prob.mz
        P.n1, P.n2, P.n3 = prob.n1, prob.n2, prob.n3
        P.n_overlap, P.n_ramp = prob.n_overlap, prob.n_ramp
        P.omega, P.velocity = prob.omega, prob.velocity
        P.c_sigma, P.sigma0 = prob.c_sigma, prob.sigma0
        self._P = P
        h = C.c_void_p()
        rc = fn("create")(C.byref(P), C.byref(h))
        if rc != 0:
            raise RuntimeError(f"orc3_create failed ({rc}): {fn('last_error')().decode()}")
        self.h = h
        self.n = int(fn("n_global")(h))
        nn = np.zeros(3, np.int32)
        fn("window_dims")(h, nn.ctypes.data_as(C.POINTER(C.c_int)))
        self.window = tuple(int(v) for v in nn)

    def class_info(self):
        out = []
        for c in range(self._fn("num_classes")(self.h)):
            m, nnz, pr = C.c_int(), C.c_long(), C.c_double()
            self._check(self._fn("class_info")(self.h, c, C.byref(m), C.byref(nnz), C.byref(pr)))
            out.append(dict(members=m.value, factor_nnz=nnz.value, probe_relres=pr.value,
                            backend="ldlt"))
        return out

    def class_of(self, t: int) -> int:
        return int(self._fn("class_of")(self.h, t))

    def class_solve(self, c: int, b):
        b = _cvec(b)
        x = np.empty_like(b)
        rel = C.c_double()
        self._check(self._fn("class_solve")(self.h, c, _dp(b), _dp(x), C.byref(rel)))
        return x, rel.value

    def class_matvec(self, c: int, x):
        x = _cvec(x)
        y = np.empty_like(x)
        self._check(self._fn("class_matvec")(self.h, c, _dp(x), _dp(y)))
        return y

    def tap_subdomain(self, t: int):
        nw = int(np.prod(self.window))
        rhs = np.zeros(nw, np.complex128)
        u = np.zeros(nw, np.complex128)
        act = C.c_int()
        self._check(self._fn("tap_subdomain")(self.h, t, _dp(rhs), _dp(u), C.byref(act)))
        return rhs, u, bool(act.value)


def nd_order3(nx: int, ny: int, nz: int) -> np.ndarray:
    out = np.zeros(nx * ny * nz, np.int32)
    _lib3().orc3_nd_order(nx, ny, nz, out.ctypes.data_as(C.POINTER(C.c_int)))
    return out


def direction3(d: int):
    o = np.zeros(3, np.int32)
    _lib3().orc3_direction(d, o.ctypes.data_as(C.POINTER(C.c_int)))
    return tuple(int(v) for v in o)
