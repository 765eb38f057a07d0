"""Python mirror of the 3-D entry points (include/hddm3.h) over libhddm.so.

``DdmEngine3`` carries the surface of ``DdmEngine`` (engine.py, mirroring
proj/include/helmddm/ddm.hpp:53-109) for a 3-D ``Problem3`` (BASELINE config 5):
same method names, argument meaning and errors. The reference has no 3-D code;
the math is the restatement oracle/hddm_oracle3.c. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np

from .engine import (ConfigError, DdmStats, FgmresOptions, FgmresResult, HddmError, SolveError,
                     StepRecord, _FgRes, _Stats, _is_torch, _raise, load_library, HDDM_DEVICE,
                     HDDM_HOST)
from .problems import Problem3


class _Problem3(C.Structure):
    _fields_ = [
        ("x0", C.c_double), ("y0", C.c_double), ("z0", C.c_double), ("h", C.c_double),
        ("mx", C.c_int), ("my", C.c_int), ("mz", C.c_int),
        ("n1", C.c_int), ("n2", C.c_int), ("n3", C.c_int),
        ("n_overlap", C.c_int), ("n_ramp", C.c_int),
        ("omega", C.c_double), ("velocity", C.c_double),
        ("c_sigma", C.c_double), ("sigma0", C.c_double), ("device", C.c_int),
    ]


_have3 = False


def load_library3():
    """libhddm.so with the hddm3_* signatures declared."""
    global _have3
    lib = load_library()
    if _have3:
        return lib
    P, d, dp, ip, vp = C.POINTER, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_void_p
    L = P(C.c_long)
    sigs = {
        "hddm3_last_error": (C.c_char_p, [vp]),
        "hddm3_create": (C.c_int, [P(_Problem3), P(vp)]),
        "hddm3_destroy": (None, [vp]),
        "hddm3_n_global": (C.c_long, [vp]),
        "hddm3_sigma0": (d, [vp]),
        "hddm3_factor_ms": (d, [vp]),
        "hddm3_num_subdomains": (C.c_int, [vp]),
        "hddm3_num_classes": (C.c_int, [vp]),
        "hddm3_class_of": (C.c_int, [vp, C.c_int]),
        "hddm3_class_info": (C.c_int, [vp, C.c_int, ip, L, dp]),
        "hddm3_window_dims": (C.c_int, [vp, ip]),
        "hddm3_apply_global": (C.c_int, [vp, vp, vp, C.c_int]),
        "hddm3_solve_iterative": (C.c_int, [vp, vp, d, C.c_int, C.c_int, vp, C.c_int, P(_Stats), ip,
                                            dp, dp, C.c_int, ip]),
        "hddm3_precondition": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, P(_Stats)]),
        "hddm3_fgmres": (C.c_int, [vp, vp, vp, d, C.c_int, C.c_int, C.c_int, C.c_int, P(_FgRes), dp,
                                   C.c_int, P(_Stats)]),
        "hddm3_fgmres_z": (C.c_int, [vp, C.c_int, vp, C.c_int]),
        "hddm3_tap_subdomain": (C.c_int, [vp, C.c_int, dp, dp, ip]),
        "hddm3_class_solve": (C.c_int, [vp, C.c_int, dp, dp, dp]),
        "hddm3_symbolic_stats": (C.c_int, [C.c_int, C.c_int, C.c_int, L, L, ip, ip, L]),
        "hddm3_nd_order": (C.c_int, [C.c_int, C.c_int, C.c_int, ip]),
        "hddm3_footprint": (C.c_int, [vp, L, L, L]),
        "hddm3_time_solve": (C.c_int, [vp, C.c_int, dp]),
        "hddm3_solve_launches": (C.c_int, [vp]),
        "hddm3_refine_stats": (C.c_int, [vp, dp, ip]),
        "hddm3_set_timing": (C.c_int, [vp, C.c_int]),
        "hddm3_launch_count": (C.c_longlong, [vp]),
        "hddm3_stream": (vp, [vp]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _have3 = True
    return lib


def nd_order3(nx: int, ny: int, nz: int) -> np.ndarray:
    """The 3-D elimination order as the engine computes it (host only)."""
    lib = load_library3()
    out = np.zeros(nx * ny * nz, np.int32)
    rc = lib.hddm3_nd_order(nx, ny, nz, out.ctypes.data_as(C.POINTER(C.c_int)))
    if rc:
        _raise(rc, lib.hddm3_last_error(None).decode())
    return out


def symbolic_stats3(nx: int, ny: int, nz: int) -> dict:
    """Host-only symbolic analysis of a 3-D window (no GPU)."""
    lib = load_library3()
    a, b, e = C.c_long(), C.c_long(), C.c_long()
    c, d = C.c_int(), C.c_int()
    rc = lib.hddm3_symbolic_stats(nx, ny, nz, C.byref(a), C.byref(b), C.byref(c), C.byref(d),
                                  C.byref(e))
    if rc:
        _raise(rc, lib.hddm3_last_error(None).decode())
    return dict(nnz_ref=a.value, stored=b.value, supernodes=c.value, height=d.value,
                front_words=e.value)


class DdmEngine3:
    """DdmEngine's surface for a 3-D problem on one B200."""

    def __init__(self, prob: Problem3, device: int = 0):
        self.lib = load_library3()
        self.prob = prob
        P = _Problem3()
        P.x0, P.y0, P.z0, P.h = prob.x0, prob.y0, prob.z0, prob.h
        P.mx, P.my, P.mz = prob.mx, prob.my, prob.mz
        P.n1, P.n2, P.n3 = prob.n1, prob.n2, prob.n3
        P.n_overlap, P.n_ramp = prob.n_overlap, prob.n_ramp
        P.omega, P.velocity = prob.omega, prob.velocity
        P.c_sigma, P.sigma0, P.device = prob.c_sigma, prob.sigma0, device
        h = C.c_void_p()
        rc = self.lib.hddm3_create(C.byref(P), C.byref(h))
        if rc != 0:
            _raise(rc, self.lib.hddm3_last_error(None).decode())
        self.h = h
        self.device = device
        self.n = int(self.lib.hddm3_n_global(h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.hddm3_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc: int):
        if rc != 0:
            _raise(rc, self.lib.hddm3_last_error(self.h).decode())

    # -- accessors
    def n_global(self) -> int:
        return self.n

    def sigma0(self) -> float:
        return float(self.lib.hddm3_sigma0(self.h))

    def factor_ms(self) -> float:
        return float(self.lib.hddm3_factor_ms(self.h))

    def num_subdomains(self) -> int:
        return int(self.lib.hddm3_num_subdomains(self.h))

    def class_of(self, t: int) -> int:
        return int(self.lib.hddm3_class_of(self.h, t))

    def class_info(self):
        out = []
        for c in range(self.lib.hddm3_num_classes(self.h)):
            m, nnz, pr = C.c_int(), C.c_long(), C.c_double()
            self._check(self.lib.hddm3_class_info(self.h, c, C.byref(m), C.byref(nnz), C.byref(pr)))
            out.append(dict(members=m.value, factor_nnz=nnz.value, probe_relres=pr.value,
                            backend="ldlt"))
        return out

    def footprint(self):
        s, r, b = C.c_long(), C.c_long(), C.c_long()
        self._check(self.lib.hddm3_footprint(self.h, C.byref(s), C.byref(r), C.byref(b)))
        return dict(stored_values_per_class=s.value, ref_nnz_per_class=r.value,
                    device_bytes_in_use=b.value)

    def window_dims(self) -> Tuple[int, int, int]:
        nn = np.zeros(3, np.int32)
        self._check(self.lib.hddm3_window_dims(self.h, nn.ctypes.data_as(C.POINTER(C.c_int))))
        return tuple(int(v) for v in nn)

    # -- argument marshalling (as DdmEngine._io)
    def _io(self, a, writable=False):
        if _is_torch(a):
            import torch
            if not a.is_cuda or a.dtype != torch.complex128 or not a.is_contiguous():
                raise ConfigError("device vectors must be contiguous complex128 CUDA tensors")
            if a.numel() != self.n:
                raise SolveError("source vector size mismatch")
            return C.c_void_p(a.data_ptr()), HDDM_DEVICE, a
        arr = np.asarray(a)
        if arr.dtype != np.complex128 or not arr.flags.c_contiguous or (writable and not arr.flags.writeable):
            if writable:
                raise ConfigError("output arrays must be writable C-contiguous complex128")
            arr = np.ascontiguousarray(arr, dtype=np.complex128)
        if arr.size != self.n:
            raise SolveError("source vector size mismatch")
        return C.c_void_p(arr.ctypes.data), HDDM_HOST, arr

    def _out_like(self, a):
        if _is_torch(a):
            import torch
            return torch.empty_like(a)
        return np.empty(self.n, np.complex128)

    # -- DdmEngine API
    def apply_global(self, u, out=None):
        pu, mk, keep = self._io(u)
        out = self._out_like(u) if out is None else out
        po, mk2, keep2 = self._io(out, writable=True)
        if mk != mk2:
            raise ConfigError("u and out must live in the same memory")
        self._check(self.lib.hddm3_apply_global(self.h, pu, po, mk))
        return out

    def solve_iterative(self, f, tol: float, max_steps: int, stats: Optional[DdmStats] = None,
                        check_every: int = 1):
        pf, mk, keep = self._io(f)
        out = self._out_like(f)
        po, _, keep2 = self._io(out, writable=True)
        st = _Stats()
        cap = max(max_steps, 1) + 1
        hs = np.zeros(cap, np.int32)
        hr = np.zeros(cap, np.float64)
        hm = np.zeros(cap, np.float64)
        hl = C.c_int()
        dp = C.POINTER(C.c_double)
        self._check(self.lib.hddm3_solve_iterative(
            self.h, pf, tol, max_steps, check_every, po, mk, C.byref(st),
            hs.ctypes.data_as(C.POINTER(C.c_int)), hr.ctypes.data_as(dp), hm.ctypes.data_as(dp),
            cap, C.byref(hl)))
        if stats is not None:
            stats.steps, stats.solves, stats.skipped = st.steps, st.solves, st.skipped
            stats.relres, stats.converged = st.relres, bool(st.converged)
            stats.factor_ms, stats.sweep_ms = st.factor_ms, st.sweep_ms
            stats.history = [StepRecord(int(hs[i]), float(hr[i]), float(hm[i]))
                             for i in range(min(hl.value, cap))]
        return out

    def precondition(self, r, ksteps: int, stats: Optional[DdmStats] = None, out=None):
        pr, mk, keep = self._io(r)
        z = self._out_like(r) if out is None else out
        pz, mk2, keep2 = self._io(z, writable=True)
        if mk != mk2:
            raise ConfigError("r and out must live in the same memory")
        st = _Stats()
        if stats is not None:
            st.solves, st.skipped, st.sweep_ms = stats.solves, stats.skipped, stats.sweep_ms
        self._check(self.lib.hddm3_precondition(self.h, pr, pz, ksteps, mk, C.byref(st)))
        if stats is not None:
            stats.solves, stats.skipped, stats.sweep_ms = st.solves, st.skipped, st.sweep_ms
            stats.factor_ms = st.factor_ms
        return z

    def fgmres(self, b, opt: FgmresOptions, ksteps: int, pstats: Optional[DdmStats] = None):
        pb, mk, keep = self._io(b)
        x = self._out_like(b)
        px, _, keep2 = self._io(x, writable=True)
        res = _FgRes()
        hist = np.zeros(max(opt.max_iters, 1), np.float64)
        st = _Stats()
        if pstats is not None:
            st.solves, st.skipped, st.sweep_ms = pstats.solves, pstats.skipped, pstats.sweep_ms
        self._check(self.lib.hddm3_fgmres(
            self.h, pb, px, opt.tol, opt.max_iters, opt.restart, ksteps, mk, C.byref(res),
            hist.ctypes.data_as(C.POINTER(C.c_double)), len(hist), C.byref(st)))
        if pstats is not None:
            pstats.solves, pstats.skipped, pstats.sweep_ms = st.solves, st.skipped, st.sweep_ms
            pstats.factor_ms = st.factor_ms
        r = FgmresResult(res.iters, bool(res.converged), res.relres, res.true_relres,
                         list(hist[:res.iters]), res.wall_ms)
        return x, r

    # -- taps
    def fgmres_z(self, j: int) -> np.ndarray:
        z = np.empty(self.n, np.complex128)
        self._check(self.lib.hddm3_fgmres_z(self.h, j, C.c_void_p(z.ctypes.data), HDDM_HOST))
        return z

    def tap_subdomain(self, t: int):
        nw = int(np.prod(self.window_dims()))
        rhs = np.zeros(nw, np.complex128)
        u = np.zeros(nw, np.complex128)
        act = C.c_int()
        dp = C.POINTER(C.c_double)
        self._check(self.lib.hddm3_tap_subdomain(self.h, t, rhs.ctypes.data_as(dp),
                                                 u.ctypes.data_as(dp), C.byref(act)))
        return rhs, u, bool(act.value)

    def class_solve(self, c: int, b):
        b = np.ascontiguousarray(b, np.complex128)
        x = np.empty_like(b)
        rel = C.c_double()
        dp = C.POINTER(C.c_double)
        self._check(self.lib.hddm3_class_solve(self.h, c, b.ctypes.data_as(dp),
                                               x.ctypes.data_as(dp), C.byref(rel)))
        return x, rel.value

    def refine_stats(self):
        m, n = C.c_double(), C.c_int()
        self._check(self.lib.hddm3_refine_stats(self.h, C.byref(m), C.byref(n)))
        return m.value, n.value

    def time_solve(self, reps: int = 10) -> float:
        ms = C.c_double()
        self._check(self.lib.hddm3_time_solve(self.h, reps, C.byref(ms)))
        return ms.value

    def solve_launches(self) -> int:
        return int(self.lib.hddm3_solve_launches(self.h))

    def set_timing(self, on: bool):
        self._check(self.lib.hddm3_set_timing(self.h, 1 if on else 0))

    def launch_count(self) -> int:
        return int(self.lib.hddm3_launch_count(self.h))

    def stream_handle(self) -> int:
        return int(self.lib.hddm3_stream(self.h) or 0)
