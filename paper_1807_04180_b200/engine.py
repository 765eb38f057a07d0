"""Python mirror of the reference's DDM entry points over the C-ABI (libhddm.so).

``DdmEngine`` mirrors ``helmddm::DdmEngine`` (proj/include/helmddm/ddm.hpp:53-109)
and ``DdmEngine.fgmres`` mirrors ``fgmres`` wired as proj/src/cli.cpp:210-228
(A = apply_global, M = precondition(K)). Same names, argument meaning and error
behaviour: ``ConfigError`` / ``SolveError`` are raised for the C codes 2 / 3
(proj/include/helmddm/types.hpp:58-66, cli.cpp:453-469).

Arrays: numpy complex128 vectors of ``n_global`` entries (host memory), or
torch complex128 CUDA tensors on the engine's device (device memory, no copies).
There is no CPU fallback: a missing library or CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from .problems import Problem

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HDDM_LIB") or os.path.join(HERE, "libhddm.so")

HDDM_HOST, HDDM_DEVICE = 0, 1


class ConfigError(RuntimeError):
    """helmddm::ConfigError (types.hpp:58-60)."""


class SolveError(RuntimeError):
    """helmddm::SolveError (types.hpp:61-63)."""


class HddmError(RuntimeError):
    """Any other failure (CUDA error, domain error)."""


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
        ("lens_amp", C.c_double), ("lens_xc", C.c_double), ("lens_yc", C.c_double),
        ("lens_w", C.c_double), ("device", C.c_int),
        ("has_box", C.c_int), ("box_x0", C.c_double), ("box_x1", C.c_double),
        ("box_y0", C.c_double), ("box_y1", C.c_double), ("margin", C.c_double),
    ]


class _Stats(C.Structure):
    _fields_ = [("steps", C.c_int), ("solves", C.c_long), ("skipped", C.c_long),
                ("relres", C.c_double), ("converged", C.c_int),
                ("factor_ms", C.c_double), ("sweep_ms", C.c_double)]


class _FgRes(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("relres", C.c_double),
                ("true_relres", C.c_double), ("wall_ms", C.c_double)]


@dataclass
class StepRecord:
    """helmddm::StepRecord (ddm.hpp:24-28)."""
    step: int
    relres: float
    wall_ms: float


@dataclass
class DdmStats:
    """helmddm::DdmStats (ddm.hpp:30-39)."""
    steps: int = 0
    solves: int = 0
    skipped: int = 0
    relres: float = -1.0
    converged: bool = False
    factor_ms: float = 0.0
    sweep_ms: float = 0.0
    history: List[StepRecord] = field(default_factory=list)


@dataclass
class FgmresOptions:
    """helmddm::FgmresOptions (krylov.hpp:11-15)."""
    tol: float = 1e-6
    max_iters: int = 200
    restart: int = 0


@dataclass
class FgmresResult:
    """helmddm::FgmresResult (krylov.hpp:17-25)."""
    iters: int = 0
    converged: bool = False
    relres: float = -1.0
    true_relres: float = -1.0
    history: List[float] = field(default_factory=list)
    wall_ms: float = 0.0


_lib = None
HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_int)  # hddm_step_hook
_OPTIONAL = {"hddm_fgmres_z", "hddm_solver_desc"}


def load_library(path: str = LIB_PATH):
    """Load libhddm.so (built by __graft_entry__.build()). Raises if missing:
    the product path has no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise HddmError(f"{path} not built; run __graft_entry__.build()")
    lib = C.CDLL(path)
    P, d, dp, ip, vp = C.POINTER, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_void_p
    sigs = {
        "hddm_last_error": (C.c_char_p, [vp]),
        "hddm_create": (C.c_int, [P(_Problem), P(vp)]),
        "hddm_destroy": (None, [vp]),
        "hddm_n_global": (C.c_long, [vp]),
        "hddm_sigma0": (d, [vp]),
        "hddm_factor_ms": (d, [vp]),
        "hddm_num_subdomains": (C.c_int, [vp]),
        "hddm_num_classes": (C.c_int, [vp]),
        "hddm_class_info": (C.c_int, [vp, C.c_int, ip, P(C.c_long), dp, ip]),
        "hddm_class_of": (C.c_int, [vp, C.c_int]),
        "hddm_apply_global": (C.c_int, [vp, vp, vp, C.c_int]),
        "hddm_solve_iterative": (C.c_int, [vp, vp, d, C.c_int, C.c_int, vp, C.c_int,
                                           P(_Stats), ip, dp, dp, C.c_int, ip]),
        "hddm_precondition": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, P(_Stats)]),
        "hddm_fgmres": (C.c_int, [vp, vp, vp, d, C.c_int, C.c_int, C.c_int, C.c_int,
                                  P(_FgRes), dp, C.c_int, P(_Stats)]),
        "hddm_fgmres_z": (C.c_int, [vp, C.c_int, vp, C.c_int]),
        "hddm_tap_subdomain": (C.c_int, [vp, C.c_int, dp, dp, ip]),
        "hddm_class_solve": (C.c_int, [vp, C.c_int, dp, dp, dp]),
        "hddm_window_dims": (C.c_int, [vp, ip, ip]),
        "hddm_nd_order": (C.c_int, [C.c_int, C.c_int, ip]),
        "hddm_footprint": (C.c_int, [vp, P(C.c_long), P(C.c_long), P(C.c_long)]),
        "hddm_symbolic_stats": (C.c_int, [C.c_int, C.c_int, P(C.c_long), P(C.c_long), ip, ip]),
        "hddm_fwd_entries": (C.c_int, [vp, P(C.c_longlong), P(C.c_longlong)]),
        "hddm_set_timing": (C.c_int, [vp, C.c_int]),
        "hddm_stage_times": (C.c_int, [vp, dp, P(C.c_longlong), C.c_int, ip]),
        "hddm_launch_count": (C.c_longlong, [vp]),
        "hddm_refine_stats": (C.c_int, [vp, dp, ip]),
        "hddm_time_solve": (C.c_int, [vp, C.c_int, dp]),
        "hddm_tune_fwd_shape": (C.c_int, [vp, C.c_int, C.c_int, C.c_int]),
        "hddm_solve_launches": (C.c_int, [vp]),
        "hddm_time_kernel": (C.c_int, [vp, C.c_int, C.c_int, dp]),
        "hddm_stage_name": (C.c_char_p, [C.c_int]),
        "hddm_stream": (vp, [vp]),
        "hddm_set_owned": (C.c_int, [vp, ip]),
        "hddm_precondition_begin": (C.c_int, [vp, vp, C.c_int]),
        "hddm_step": (C.c_int, [vp, C.c_int]),
        "hddm_halo_pack": (C.c_int, [vp, C.c_int, ip, C.c_int, dp, ip]),
        "hddm_halo_unpack": (C.c_int, [vp, C.c_int, ip, C.c_int, dp, ip]),
        "hddm_precondition_end": (C.c_int, [vp, vp, C.c_int, P(_Stats)]),
        "hddm_set_step_hook": (C.c_int, [vp, HOOK, vp]),
        "hddm_assembled": (C.c_int, [vp, dp, C.c_int]),
        "hddm_solver_desc": (C.c_char_p, [vp]),
    }
    for name, (res, args) in sigs.items():
        if name in _OPTIONAL and not hasattr(lib, name):
            continue  # an older build (tools/ comparisons only)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _raise(rc: int, msg: str):
    if rc == 2:
        raise ConfigError(msg)
    if rc == 3:
        raise SolveError(msg)
    raise HddmError(msg)


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def nd_order(nx: int, ny: int) -> np.ndarray:
    """grid_nd_order (proj/src/sparse.cpp:42-57) as computed by the engine."""
    lib = load_library()
    out = np.zeros(nx * ny, np.int32)
    lib.hddm_nd_order(nx, ny, out.ctypes.data_as(C.POINTER(C.c_int)))
    return out


def symbolic_stats(nx: int, ny: int) -> dict:
    """Host-only symbolic analysis (no GPU): reference nnz, stored entries."""
    lib = load_library()
    a, b, c, d = C.c_long(), C.c_long(), C.c_int(), C.c_int()
    rc = lib.hddm_symbolic_stats(nx, ny, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
    if rc:
        _raise(rc, lib.hddm_last_error(None).decode())
    return dict(nnz_ref=a.value, stored=b.value, supernodes=c.value, height=d.value)


class DdmEngine:
    """helmddm::DdmEngine on one B200 (ddm.hpp:53-109)."""

    def __init__(self, prob: Problem, device: int = 0):
        self.lib = load_library()
        self.prob = prob
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
        dp = C.POINTER(C.c_double)
        P.layer_ylo = self._ylo.ctypes.data_as(dp)
        P.layer_yhi = self._yhi.ctypes.data_as(dp)
        P.layer_c = self._c.ctypes.data_as(dp)
        P.c_sigma, P.sigma0, P.threads = prob.c_sigma, prob.sigma0, 1
        P.lens_amp, P.lens_xc, P.lens_yc, P.lens_w = prob.lens
        P.device = device
        h = C.c_void_p()
        rc = self.lib.hddm_create(C.byref(P), C.byref(h))
        if rc != 0:
            _raise(rc, self.lib.hddm_last_error(None).decode())
        self.h = h
        self.device = device
        self.n = int(self.lib.hddm_n_global(h))

    # -- lifetime
    def close(self):
        if getattr(self, "h", None):
            self.lib.hddm_destroy(self.h)
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
            _raise(rc, self.lib.hddm_last_error(self.h).decode())

    # -- accessors (ddm.hpp:57-63)
    def n_global(self) -> int:
        return self.n

    def sigma0(self) -> float:
        return float(self.lib.hddm_sigma0(self.h))

    def factor_ms(self) -> float:
        return float(self.lib.hddm_factor_ms(self.h))

    def num_subdomains(self) -> int:
        return int(self.lib.hddm_num_subdomains(self.h))

    def class_of(self, t: int) -> int:
        return int(self.lib.hddm_class_of(self.h, t))

    def class_info(self):
        out = []
        for c in range(self.lib.hddm_num_classes(self.h)):
            m, nnz, pr, ld = C.c_int(), C.c_long(), C.c_double(), C.c_int()
            self._check(self.lib.hddm_class_info(self.h, c, C.byref(m), C.byref(nnz),
                                                 C.byref(pr), C.byref(ld)))
            out.append(dict(members=m.value, factor_nnz=nnz.value, probe_relres=pr.value,
                            backend="ldlt" if ld.value else "lu"))
        return out

    def footprint(self):
        s, r, b = C.c_long(), C.c_long(), C.c_long()
        self._check(self.lib.hddm_footprint(self.h, C.byref(s), C.byref(r), C.byref(b)))
        return dict(stored_values_per_class=s.value, ref_nnz_per_class=r.value,
                    device_bytes_in_use=b.value)

    # -- argument marshalling
    def _io(self, a, writable=False):
        """(pointer, memkind, keepalive) for a vector argument."""
        if _is_torch(a):
            import torch
            if not a.is_cuda or a.dtype != torch.complex128 or not a.is_contiguous():
                raise ConfigError("device vectors must be contiguous complex128 CUDA tensors")
            if a.numel() != self.n:
                raise SolveError("source vector size mismatch")
            return C.c_void_p(a.data_ptr()), HDDM_DEVICE, a
        arr = np.asarray(a)
        if arr.dtype != np.complex128 or not arr.flags.c_contiguous or (writable and not arr.flags.writeable):
            if writable:  # results must land in the caller's array, not in a copy
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
        """out = L u on the global window (ddm.hpp:66)."""
        pu, mk, keep = self._io(u)
        out = self._out_like(u) if out is None else out
        po, mk2, keep2 = self._io(out, writable=True)
        if mk != mk2:
            raise ConfigError("u and out must live in the same memory")
        self._check(self.lib.hddm_apply_global(self.h, pu, po, mk))
        return out

    def solve_iterative(self, f, tol: float, max_steps: int, stats: Optional[DdmStats] = None,
                        check_every: int = 1):
        """Sweeps until relres <= tol or max_steps (ddm.hpp:72-74); returns the
        assembled global field and fills ``stats``."""
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
        self._check(self.lib.hddm_solve_iterative(
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
        """z = M(r) with K sweeps (ddm.hpp:78); counts accumulate into stats."""
        pr, mk, keep = self._io(r)
        z = self._out_like(r) if out is None else out
        pz, mk2, keep2 = self._io(z, writable=True)
        if mk != mk2:
            raise ConfigError("r and out must live in the same memory")
        st = _Stats()
        if stats is not None:
            st.solves, st.skipped, st.sweep_ms = stats.solves, stats.skipped, stats.sweep_ms
        self._check(self.lib.hddm_precondition(self.h, pr, pz, ksteps, mk, C.byref(st)))
        if stats is not None:
            stats.solves, stats.skipped, stats.sweep_ms = st.solves, st.skipped, st.sweep_ms
            stats.factor_ms = st.factor_ms
        return z

    def fgmres(self, b, opt: FgmresOptions, ksteps: int, pstats: Optional[DdmStats] = None):
        """fgmres(n, A=apply_global, M=precondition(K), b, x, opt) as
        cli.cpp:210-228 wires it; device-resident. Returns (x, FgmresResult)."""
        pb, mk, keep = self._io(b)
        x = self._out_like(b)
        px, _, keep2 = self._io(x, writable=True)
        res = _FgRes()
        hist = np.zeros(max(opt.max_iters, 1), np.float64)
        st = _Stats()
        if pstats is not None:
            st.solves, st.skipped, st.sweep_ms = pstats.solves, pstats.skipped, pstats.sweep_ms
        self._check(self.lib.hddm_fgmres(
            self.h, pb, px, opt.tol, opt.max_iters, opt.restart, ksteps, mk, C.byref(res),
            hist.ctypes.data_as(C.POINTER(C.c_double)), len(hist), C.byref(st)))
        if pstats is not None:
            pstats.solves, pstats.skipped, pstats.sweep_ms = st.solves, st.skipped, st.sweep_ms
            pstats.factor_ms = st.factor_ms
        r = FgmresResult(res.iters, bool(res.converged), res.relres, res.true_relres,
                         list(hist[:res.iters]), res.wall_ms)
        return x, r

    # -- parity / measurement taps
    def fgmres_z(self, j: int) -> np.ndarray:
        """Z_j = M(V_j) of the last FGMRES restart cycle (krylov.cpp:59-63)."""
        z = np.empty(self.n, np.complex128)
        self._check(self.lib.hddm_fgmres_z(self.h, j, C.c_void_p(z.ctypes.data), HDDM_HOST))
        return z

    def window_dims(self) -> Tuple[int, int]:
        nx, ny = C.c_int(), C.c_int()
        self._check(self.lib.hddm_window_dims(self.h, C.byref(nx), C.byref(ny)))
        return nx.value, ny.value

    def tap_subdomain(self, t: int):
        nx, ny = self.window_dims()
        rhs = np.zeros(nx * ny, np.complex128)
        u = np.zeros(nx * ny, np.complex128)
        act = C.c_int()
        dp = C.POINTER(C.c_double)
        self._check(self.lib.hddm_tap_subdomain(self.h, t, rhs.ctypes.data_as(dp),
                                                u.ctypes.data_as(dp), C.byref(act)))
        return rhs, u, bool(act.value)

    def class_solve(self, c: int, b):
        b = np.ascontiguousarray(b, np.complex128)
        x = np.empty_like(b)
        rel = C.c_double()
        dp = C.POINTER(C.c_double)
        self._check(self.lib.hddm_class_solve(self.h, c, b.ctypes.data_as(dp),
                                              x.ctypes.data_as(dp), C.byref(rel)))
        return x, rel.value

    def set_timing(self, on: bool):
        self._check(self.lib.hddm_set_timing(self.h, 1 if on else 0))

    def stage_times(self):
        """{stage: (total device ms, number of timed instances)} since set_timing."""
        buf = np.zeros(16, np.float64)
        cnt = np.zeros(16, np.int64)
        n = C.c_int()
        self._check(self.lib.hddm_stage_times(self.h, buf.ctypes.data_as(C.POINTER(C.c_double)),
                                              cnt.ctypes.data_as(C.POINTER(C.c_longlong)), 16,
                                              C.byref(n)))
        return {self.lib.hddm_stage_name(i).decode(): (float(buf[i]), int(cnt[i]))
                for i in range(n.value)}

    def refine_stats(self):
        """(max local-solve relres, number of solves above 1e-11) of the last call."""
        m, n = C.c_double(), C.c_int()
        self._check(self.lib.hddm_refine_stats(self.h, C.byref(m), C.byref(n)))
        return m.value, n.value

    def fwd_entries(self):
        """(full, sparse-RHS) factor entries of one class's forward sweep."""
        a, b = C.c_longlong(), C.c_longlong()
        self._check(self.lib.hddm_fwd_entries(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def time_solve(self, reps: int = 10) -> float:
        """Average device ms of one batched solve stage (steady state)."""
        ms = C.c_double()
        self._check(self.lib.hddm_time_solve(self.h, reps, C.byref(ms)))
        return ms.value

    def tune_fwd_shape(self, which: int, level: int, lanes: int):
        """Tuning aid: lane shape of a steady-state forward level (hddm_tune_fwd_shape)."""
        self._check(self.lib.hddm_tune_fwd_shape(self.h, which, level, lanes))

    def time_kernel(self, which: str, reps: int = 20) -> float:
        """Device ms of one launch of a step stage kernel (transfer / check / accumulate)
        on the last sweep's state (hddm_time_kernel)."""
        idx = {"transfer": 0, "check": 1, "accumulate": 2}[which]
        ms = C.c_double()
        self._check(self.lib.hddm_time_kernel(self.h, idx, reps, C.byref(ms)))
        return ms.value

    def solve_launches(self) -> int:
        return int(self.lib.hddm_solve_launches(self.h))

    def launch_count(self) -> int:
        return int(self.lib.hddm_launch_count(self.h))

    def solver_desc(self) -> str:
        return self.lib.hddm_solver_desc(self.h).decode()

    def stream_handle(self) -> int:
        return int(self.lib.hddm_stream(self.h) or 0)

    # -- sharded runs (hddm.h "sharded runs"; driven by shard.py)
    def set_owned(self, owned):
        """Subdomains this engine solves (None: all)."""
        if owned is None:
            self._check(self.lib.hddm_set_owned(self.h, None))
            return
        o = np.ascontiguousarray(owned, np.int32)
        self._check(self.lib.hddm_set_owned(self.h, o.ctypes.data_as(C.POINTER(C.c_int))))

    def precondition_begin(self, r):
        pr, mk, keep = self._io(r)
        self._check(self.lib.hddm_precondition_begin(self.h, pr, mk))
        self._begin_kind = mk

    def step(self, s: int):
        self._check(self.lib.hddm_step(self.h, s))

    def halo_pack(self, s: int, ts):
        """(solutions [len(ts), n_w] complex, zero flags) of subdomains ts after step s."""
        ts = np.ascontiguousarray(ts, np.int32)
        nw = int(np.prod(self.window_dims()))
        buf = np.empty((len(ts), nw), np.complex128)
        flags = np.empty(len(ts), np.int32)
        ip = C.POINTER(C.c_int)
        self._check(self.lib.hddm_halo_pack(self.h, s, ts.ctypes.data_as(ip), len(ts),
                                            buf.ctypes.data_as(C.POINTER(C.c_double)),
                                            flags.ctypes.data_as(ip)))
        return buf, flags

    def halo_unpack(self, s: int, ts, buf, flags):
        ts = np.ascontiguousarray(ts, np.int32)
        buf = np.ascontiguousarray(buf, np.complex128)
        flags = np.ascontiguousarray(flags, np.int32)
        ip = C.POINTER(C.c_int)
        self._check(self.lib.hddm_halo_unpack(self.h, s, ts.ctypes.data_as(ip), len(ts),
                                              buf.ctypes.data_as(C.POINTER(C.c_double)),
                                              flags.ctypes.data_as(ip)))

    def precondition_end(self, stats: Optional[DdmStats] = None):
        """This engine's assembled field (numpy, host) after the sharded sweeps."""
        z = np.empty(self.n, np.complex128)
        st = _Stats()
        self._check(self.lib.hddm_precondition_end(self.h, C.c_void_p(z.ctypes.data), HDDM_HOST,
                                                   C.byref(st)))
        if stats is not None:
            stats.solves += st.solves
            stats.skipped += st.skipped
        return z

    def set_step_hook(self, fn):
        """fn(stage, s) after every DDM step (stage 1) and every preconditioner
        application (stage 2) of a host-driven FGMRES (sharded runs); None clears it."""
        self._hook = HOOK(lambda user, stage, s: fn(stage, s)) if fn else C.cast(None, HOOK)
        self._check(self.lib.hddm_set_step_hook(self.h, self._hook, None))

    def assembled(self, values=None):
        """Read (values None) or write the engine's assembled field (host numpy)."""
        dp = C.POINTER(C.c_double)
        if values is None:
            a = np.empty(self.n, np.complex128)
            self._check(self.lib.hddm_assembled(self.h, a.ctypes.data_as(dp), 0))
            return a
        a = np.ascontiguousarray(values, np.complex128)
        self._check(self.lib.hddm_assembled(self.h, a.ctypes.data_as(dp), 1))

