"""`helmddm` command line on the B200 engine.

Mirrors the reference CLI (proj/src/cli.cpp, config.cpp, io.cpp, medium.cpp)
so `helmddm solve <config>` runs unchanged on the GPU path:

  python -m paper_1807_04180_b200.cli solve run.cfg [--override key=value] [--quiet]
  python -m paper_1807_04180_b200.cli render run_field.hdmf out.ppm

* config: the reference's `key = value` format, the same keys, defaults,
  validation and messages (config.cpp:49-151); `--override` pairs apply after
  the file (config.cpp:155-170);
* setup: make_setup (config.cpp:180-228) -- cell counts snapped to the
  partition, equal layer bands or the default 5-band ladder, source at the
  domain centre unless placed, k at the source (medium.cpp:31-50);
* source: sample_source (medium.cpp:52-73) on the global window;
* modes: `solver.mode = ddm` -> DdmEngine.solve_iterative (cli.cpp:170-205),
  `fgmres` -> device FGMRES preconditioned by K = precond.k or n1 + n2 sweeps
  (cli.cpp:207-260);
* artifacts: `<prefix>_field.hdmf` (HDMF v1, io.cpp:26-44), `<prefix>_real.ppm`
  (io.cpp:71-99), `<prefix>_resid.csv` (io.cpp:101-114), `<prefix>_stats.txt`
  (cli.cpp:97-135);
* exit codes: 0 ok, 2 config error, 3 solver error / not converged, 4 io error,
  1 other (cli.cpp:453-469).

The reference's `direct` and `convergence` commands factor the whole global
system on the host (its oracle, not the DDM hot path); this CLI reports them
as unsupported (exit 2). In fgmres mode the device-resident FGMRES does not
timestamp single iterations: `wall_ms` in the residual CSV is the run's mean
time per iteration.
"""
from __future__ import annotations

import math
import os
import struct
import sys
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .engine import ConfigError, DdmEngine, DdmStats, FgmresOptions, HddmError, SolveError
from .problems import MEDIUM_CONSTANT, MEDIUM_LAYERED, Problem


class IoError(Exception):
    """helmddm::IoError (types.hpp)."""


USAGE = (
    "usage: helmddm <command> [options]\n"
    "commands:\n"
    "  solve <config>         run the mode selected by solver.mode\n"
    "  direct <config>        factor and solve the global system in one shot\n"
    "  convergence <config>   dyadic mesh refinement study\n"
    "  render <dump> <out.ppm>\n"
    "options:\n"
    "  --override key=value   set/replace a config entry (repeatable)\n"
    "  --quiet                suppress progress output\n")


# ------------------------------------------------------------------ config
@dataclass
class RunConfig:
    """helmddm::RunConfig (config.hpp:14-47): defaults as the reference."""
    domain: Tuple[float, float, float, float] = (0.0, 1.0, 0.0, 1.0)  # x0 x1 y0 y1
    freq: float = 0.0
    medium_type: str = "constant"
    velocity: float = 1.0
    layer_velocities: List[float] = field(default_factory=list)
    grid_h: float = 0.0
    grid_ppw: float = 0.0
    n1: int = 1
    n2: int = 1
    n_ramp: int = 20
    n_overlap: int = 10
    c_sigma: float = 25.0
    sigma0: float = 0.0
    source_type: str = "gaussian"
    source_x: float = 0.0
    source_y: float = 0.0
    source_at_center: bool = True
    mode: str = "ddm"
    tol: float = 1e-8
    max_steps: int = 200
    check_every: int = 1
    precond_k: int = 0
    krylov_tol: float = 1e-8
    krylov_max_iter: int = 200
    krylov_restart: int = 0
    prefix: str = "out"
    threads: int = 1
    conv_levels: int = 3
    conv_ref: str = "direct"
    sparse_backend: str = "auto"


def _num(key: str, v: str) -> float:
    """parse_num (config.cpp:19-27): std::stod of the whole (trimmed) value --
    decimal, hex-float, inf/nan spellings; anything left over is an error."""
    s = v.strip(" \t\r\n")
    try:
        if "_" in s:
            raise ValueError
        return float(s)
    except ValueError:
        pass
    try:
        return float.fromhex(s)
    except ValueError:
        raise ConfigError(f"bad numeric value for '{key}': {v}") from None


def _int(key: str, v: str) -> int:
    x = _num(key, v)
    i = int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))  # lround
    if float(i) != x:
        raise ConfigError(f"expected integer for '{key}'")
    return i


def _list(key: str, v: str) -> List[float]:
    out = [_num(key, item.strip()) for item in v.split(",") if item.strip()]
    if not out:
        raise ConfigError(f"empty list for '{key}'")
    return out


def _apply_pair(c: RunConfig, key: str, val: str) -> None:
    """apply_pair (config.cpp:49-88)."""
    x0, x1, y0, y1 = c.domain
    if key == "domain.x0": c.domain = (_num(key, val), x1, y0, y1)
    elif key == "domain.x1": c.domain = (x0, _num(key, val), y0, y1)
    elif key == "domain.y0": c.domain = (x0, x1, _num(key, val), y1)
    elif key == "domain.y1": c.domain = (x0, x1, y0, _num(key, val))
    elif key == "freq": c.freq = _num(key, val)
    elif key == "medium.type": c.medium_type = val
    elif key == "medium.velocity": c.velocity = _num(key, val)
    elif key == "medium.layers": c.layer_velocities = _list(key, val)
    elif key == "grid.h": c.grid_h = _num(key, val)
    elif key == "grid.ppw": c.grid_ppw = _num(key, val)
    elif key == "part.n1": c.n1 = _int(key, val)
    elif key == "part.n2": c.n2 = _int(key, val)
    elif key == "pml.n_ramp": c.n_ramp = _int(key, val)
    elif key == "pml.n_overlap": c.n_overlap = _int(key, val)
    elif key == "pml.c_sigma": c.c_sigma = _num(key, val)
    elif key == "pml.sigma0": c.sigma0 = _num(key, val)
    elif key == "source.type": c.source_type = val
    elif key == "source.x":
        c.source_x = _num(key, val)
        c.source_at_center = False
    elif key == "source.y":
        c.source_y = _num(key, val)
        c.source_at_center = False
    elif key == "solver.mode": c.mode = val
    elif key == "solver.tol": c.tol = _num(key, val)
    elif key == "solver.max_steps": c.max_steps = _int(key, val)
    elif key == "solver.check_every": c.check_every = _int(key, val)
    elif key == "precond.k": c.precond_k = _int(key, val)
    elif key == "krylov.tol": c.krylov_tol = _num(key, val)
    elif key == "krylov.max_iter": c.krylov_max_iter = _int(key, val)
    elif key == "krylov.restart": c.krylov_restart = _int(key, val)
    elif key == "output.prefix": c.prefix = val
    elif key == "threads": c.threads = _int(key, val)
    elif key == "conv.levels": c.conv_levels = _int(key, val)
    elif key == "conv.ref": c.conv_ref = val
    elif key == "sparse.backend": c.sparse_backend = val
    else:
        raise ConfigError(f"unknown config key: {key}")


def _check_enum(key: str, v: str, allowed: Sequence[str]) -> None:
    if v not in allowed:
        raise ConfigError(f"invalid value for {key}: {v}")


def _validate(c: RunConfig) -> None:
    """validate (config.cpp:110-151)."""
    x0, x1, y0, y1 = c.domain
    if not (x1 - x0 > 0) or not (y1 - y0 > 0):
        raise ConfigError("domain must have positive extent")
    if not (c.freq > 0):
        raise ConfigError("freq must be positive")
    _check_enum("medium.type", c.medium_type, ("constant", "layered"))
    if c.medium_type == "constant" and not (c.velocity > 0):
        raise ConfigError("medium.velocity must be positive")
    for v in c.layer_velocities:
        if not (v > 0):
            raise ConfigError("layer velocities must be positive")
    if (c.grid_h > 0) == (c.grid_ppw > 0):
        raise ConfigError("set exactly one of grid.h and grid.ppw")
    if c.grid_h < 0 or c.grid_ppw < 0:
        raise ConfigError("grid spacing parameters must be positive")
    if c.n1 < 1 or c.n2 < 1:
        raise ConfigError("part.n1/n2 must be >= 1")
    if c.n_ramp < 1:
        raise ConfigError("pml.n_ramp must be >= 1")
    if c.n_overlap < 0:
        raise ConfigError("pml.n_overlap must be >= 0")
    if not (c.c_sigma > 0) and not (c.sigma0 > 0):
        raise ConfigError("pml.c_sigma or pml.sigma0 must be positive")
    _check_enum("source.type", c.source_type, ("gaussian", "point"))
    _check_enum("solver.mode", c.mode, ("ddm", "fgmres", "direct"))
    if not (c.tol > 0) or not (c.krylov_tol > 0):
        raise ConfigError("tolerances must be positive")
    if c.max_steps < 1 or c.krylov_max_iter < 1:
        raise ConfigError("iteration limits must be >= 1")
    if c.check_every < 1:
        raise ConfigError("solver.check_every must be >= 1")
    if c.precond_k < 0:
        raise ConfigError("precond.k must be nonnegative")
    if c.krylov_restart < 0:
        raise ConfigError("krylov.restart must be >= 0")
    if c.threads < 1:
        raise ConfigError("threads must be >= 1")
    if c.conv_levels < 2:
        raise ConfigError("conv.levels must be >= 2")
    _check_enum("conv.ref", c.conv_ref, ("direct", "greens"))
    _check_enum("sparse.backend", c.sparse_backend, ("auto", "lu"))
    if not c.prefix:
        raise ConfigError("output.prefix must be nonempty")


def parse_config_text(text: str, overrides: Sequence[str] = ()) -> RunConfig:
    """parse_config_text (config.cpp:155-170): `key = value` lines, `#` comments."""
    c = RunConfig()
    for lineno, line in enumerate(text.split("\n"), start=1):
        line = line.split("#", 1)[0].strip(" \t\r\n")
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"line {lineno}: expected key = value")
        key, val = line.split("=", 1)
        key, val = key.strip(" \t\r\n"), val.strip(" \t\r\n")
        if not key:
            raise ConfigError(f"line {lineno}: empty key")
        _apply_pair(c, key, val)
    for ov in overrides:
        if "=" not in ov:
            raise ConfigError(f"override must be key=value: {ov}")
        key, val = ov.split("=", 1)
        _apply_pair(c, key.strip(" \t\r\n"), val.strip(" \t\r\n"))
    _validate(c)
    return c


def parse_config_file(path: str, overrides: Sequence[str] = ()) -> RunConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise IoError(f"cannot open config file: {path}") from None
    return parse_config_text(text, overrides)


# ------------------------------------------------------------------ setup
def default_layered(y0: float, y1: float) -> List[Tuple[float, float, float]]:
    """default_layered (medium.cpp:22-29): 5 equal bands, c = 1..2.5."""
    v = (1.00, 1.25, 1.60, 2.00, 2.50)
    dy = (y1 - y0) / 5.0
    return [(y0 + i * dy, y1 if i == 4 else y0 + (i + 1) * dy, v[i]) for i in range(5)]


def _lround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


@dataclass
class Setup:
    """helmddm::ProblemSetup (config.hpp:53-59) as a GPU-engine Problem."""
    problem: Problem
    source_kind: str
    source_x: float
    source_y: float
    k_source: float


def eval_wavenumber(prob: Problem, x: float, y: float) -> float:
    """eval_wavenumber (medium.cpp:31-50): constant / layered, y clamped to the
    interior, upper-boundary ties to the band below."""
    ix0, ix1 = prob.x0, prob.x0 + prob.mx * prob.h
    iy0, iy1 = prob.y0, prob.y0 + prob.my * prob.h
    m = (prob.n_ext + 1) * prob.h
    if x < ix0 - m or x > ix1 + m or y < iy0 - m or y > iy1 + m:
        raise ConfigError("eval_wavenumber: point outside the padded domain")
    yc = min(max(y, iy0), iy1)
    if prob.medium_kind == MEDIUM_CONSTANT:
        c = prob.velocity
    else:
        c = prob.layers[-1][2]
        for lo, hi, v in prob.layers:
            if yc <= hi:
                c = v
                break
    return prob.omega / c


def make_setup(cfg: RunConfig) -> Setup:
    """make_setup (config.cpp:180-228)."""
    x0, x1, y0, y1 = cfg.domain
    omega = 2.0 * math.pi * cfg.freq
    if cfg.medium_type == "constant":
        kind, layers, cmin = MEDIUM_CONSTANT, [], cfg.velocity
    else:
        kind = MEDIUM_LAYERED
        if not cfg.layer_velocities:
            layers = default_layered(y0, y1)
        else:
            n = len(cfg.layer_velocities)
            dy = (y1 - y0) / n
            layers = [(y0 + i * dy, y1 if i == n - 1 else y0 + (i + 1) * dy,
                       cfg.layer_velocities[i]) for i in range(n)]
        cmin = min(v for _, _, v in layers)
    h_goal = cfg.grid_h if cfg.grid_h > 0 else cmin / (cfg.freq * cfg.grid_ppw)
    mx = cfg.n1 * max(1, _lround((x1 - x0) / (h_goal * cfg.n1)))
    h = (x1 - x0) / mx
    my = cfg.n2 * max(1, _lround((y1 - y0) / (h * cfg.n2)))
    iy1 = y0 + my * h
    if kind == MEDIUM_LAYERED and not cfg.layer_velocities and abs(iy1 - y1) > 1e-12 * h:
        layers = default_layered(y0, iy1)
    prob = Problem(name="cli", mx=mx, my=my, h=h, x0=x0, y0=y0, n1=cfg.n1, n2=cfg.n2,
                   n_overlap=cfg.n_overlap, n_ramp=cfg.n_ramp, omega=omega,
                   medium_kind=kind, velocity=cfg.velocity, layers=layers,
                   c_sigma=cfg.c_sigma, sigma0=cfg.sigma0)
    sx = 0.5 * (x0 + x1) if cfg.source_at_center else cfg.source_x
    sy = 0.5 * (y0 + iy1) if cfg.source_at_center else cfg.source_y
    return Setup(prob, cfg.source_type, sx, sy, eval_wavenumber(prob, sx, sy))


def sample_source(st: Setup) -> np.ndarray:
    """sample_source (medium.cpp:52-73) on the global window, row-major x fastest."""
    prob = st.problem
    xs, ys = prob.lattice_xy()
    if st.source_kind == "point":
        ox = prob.x0 - prob.n_ext * prob.h
        oy = prob.y0 - prob.n_ext * prob.h
        p = math.ceil((st.source_x - ox) / prob.h - 0.5)
        q = math.ceil((st.source_y - oy) / prob.h - 0.5)
        f = np.zeros((prob.gny, prob.gnx), np.complex128)
        if 0 <= p < prob.gnx and 0 <= q < prob.gny:
            f[q, p] = 1.0 / (prob.h * prob.h)
        return f.ravel()
    k = st.k_source
    amp = 16.0 * k * k / (math.pi * math.pi * math.pi)
    w = 4.0 * k / math.pi
    w2 = w * w
    dx = xs - st.source_x
    dy = ys - st.source_y
    f = amp * np.exp(-w2 * (dx[None, :] * dx[None, :] + dy[:, None] * dy[:, None]))
    return f.astype(np.complex128).ravel()


# ------------------------------------------------------------------ artifacts
def write_field_dump(path: str, nx: int, ny: int, x0: float, y0: float, h: float,
                     data: np.ndarray) -> None:
    """write_field_dump (io.cpp:26-44): "HDMF", u32 version 1, u32 nx, ny,
    f64 x0, y0, h, then nx*ny complex128 (little-endian)."""
    try:
        with open(path, "wb") as f:
            f.write(b"HDMF" + struct.pack("<III", 1, nx, ny) + struct.pack("<ddd", x0, y0, h))
            f.write(np.ascontiguousarray(data, dtype="<c16").tobytes())
    except OSError:
        raise IoError(f"cannot open for writing: {path}") from None


def read_field_dump(path: str):
    """read_field_dump (io.cpp:46-69) -> (nx, ny, x0, y0, h, data)."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError:
        raise IoError(f"cannot open: {path}") from None
    if raw[:4] != b"HDMF":
        raise IoError(f"not a field dump: {path}")
    if len(raw) < 40:
        raise IoError(f"truncated field dump: {path}")
    version, nx, ny = struct.unpack("<III", raw[4:16])
    if version != 1:
        raise IoError(f"unsupported dump version in {path}")
    x0, y0, h = struct.unpack("<ddd", raw[16:40])
    n = nx * ny * 16
    if len(raw) < 40 + n:
        raise IoError(f"truncated field dump: {path}")
    if len(raw) > 40 + n:
        raise IoError(f"trailing bytes in field dump: {path}")
    data = np.frombuffer(raw[40:], dtype="<c16").astype(np.complex128)
    return nx, ny, x0, y0, h, data


def write_ppm_real(path: str, nx: int, ny: int, data: np.ndarray, vmax: float = 0.0) -> None:
    """write_ppm_real (io.cpp:71-99): red for positive, blue for negative real part."""
    re = np.real(data).astype(np.float64)
    if vmax <= 0:
        vmax = max(0.0, float(np.max(np.abs(re)))) if re.size else 0.0
    v = re / vmax if vmax > 0 else np.zeros_like(re)
    v = np.clip(v, -1.0, 1.0)
    # std::lround: halves away from zero (the argument is nonnegative here)
    pos = np.floor(255.0 * (1.0 - v) + 0.5).astype(np.uint8)
    neg = np.floor(255.0 * (1.0 + v) + 0.5).astype(np.uint8)
    rgb = np.empty((re.size, 3), np.uint8)
    ge = v >= 0
    rgb[:, 0] = np.where(ge, 255, neg)
    rgb[:, 1] = np.where(ge, pos, neg)
    rgb[:, 2] = np.where(ge, pos, 255)
    try:
        with open(path, "wb") as f:
            f.write(f"P6\n{nx} {ny}\n255\n".encode())
            f.write(rgb.tobytes())
    except OSError:
        raise IoError(f"cannot open for writing: {path}") from None


def write_resid_csv(path: str, hist: Sequence[Tuple[int, float, float]]) -> None:
    """write_resid_csv (io.cpp:101-114)."""
    try:
        with open(path, "w") as f:
            f.write("step,relres,wall_ms\n")
            for step, rel, ms in hist:
                f.write("%d,%.6e,%.3f\n" % (step, rel, ms))
    except OSError:
        raise IoError(f"cannot open for writing: {path}") from None


@dataclass
class RunArtifacts:
    """RunArtifacts (cli.cpp:80-95)."""
    mode: str = ""
    prob: Optional[Problem] = None
    sigma0: float = 0.0
    threads: int = 1
    classes: list = field(default_factory=list)
    n_ddm_iter: int = 0
    sweep_len: int = 1
    n_gmres_iter: int = 0
    precond_k: int = 0
    relres: float = -1.0
    true_relres: float = -1.0
    converged: bool = True
    factor_ms: float = 0.0
    solve_ms: float = 0.0
    total_ms: float = 0.0


def write_stats(path: str, r: RunArtifacts) -> None:
    """write_stats (cli.cpp:97-135), same keys and number formats."""
    lines = [f"mode = {r.mode}\n"]
    if r.prob is not None:
        p = r.prob
        lines.append("grid.cells = %d x %d\ngrid.h = %.9e\npartition = %d x %d\n"
                     "pml.n_ramp = %d\npml.n_overlap = %d\npml.sigma0 = %.9e\n"
                     % (p.mx, p.my, p.h, p.n1, p.n2, p.n_ramp, p.n_overlap, r.sigma0))
    lines.append(f"threads = {r.threads}\n")
    n_ldlt = sum(1 for c in r.classes if c.get("backend") == "ldlt")
    lines.append(f"factor.classes = {len(r.classes)}\n")
    lines.append(f"factor.backend.ldlt = {n_ldlt}\n")
    lines.append(f"factor.backend.lu = {len(r.classes) - n_ldlt}\n")
    lines.append(f"n_DDM_Iter = {r.n_ddm_iter}\n")
    lines.append("n_DDM_Solv = %.2f\n" % (r.n_ddm_iter / r.sweep_len))
    lines.append(f"n_GMRES_Iter = {r.n_gmres_iter}\n")
    lines.append(f"n_Local_Solv = {r.n_gmres_iter * r.precond_k}\n")
    if r.precond_k > 0:
        lines.append(f"precond.k = {r.precond_k}\n")
    lines.append("relres = %.6e\n" % r.relres)
    if r.true_relres >= 0:
        lines.append("true_relres = %.6e\n" % r.true_relres)
    lines.append("converged = %s\n" % ("yes" if r.converged else "no"))
    lines.append("factor_ms = %.1f\nsolve_ms = %.1f\ntotal_ms = %.1f\n"
                 % (r.factor_ms, r.solve_ms, r.total_ms))
    try:
        with open(path, "w") as f:
            f.write("".join(lines))
    except OSError:
        raise IoError(f"cannot open for writing: {path}") from None


def write_field_artifacts(cfg: RunConfig, prob: Problem, u: np.ndarray) -> None:
    """write_field_artifacts (cli.cpp:137-143): global window dump + image."""
    ox = prob.x0 - prob.n_ext * prob.h
    oy = prob.y0 - prob.n_ext * prob.h
    write_field_dump(cfg.prefix + "_field.hdmf", prob.gnx, prob.gny, ox, oy, prob.h, u)
    write_ppm_real(cfg.prefix + "_real.ppm", prob.gnx, prob.gny, u, 0.0)


# ------------------------------------------------------------------ runs
def _announce(quiet: bool, line: str) -> None:
    if not quiet:
        print(line, flush=True)


def _describe(p: Problem, sigma0: float) -> str:
    return "grid %dx%d cells, h=%.4e, partition %dx%d, sigma0=%.4e" % (
        p.mx, p.my, p.h, p.n1, p.n2, sigma0)


def env_threads(fallback: int) -> int:
    """env_threads (cli.cpp:63-72): HELMDDM_THREADS overrides `threads`."""
    e = os.environ.get("HELMDDM_THREADS", "")
    if not e:
        return fallback
    try:
        v = int(e, 10)
    except ValueError:
        raise ConfigError("bad HELMDDM_THREADS value") from None
    if v < 1:
        raise ConfigError("bad HELMDDM_THREADS value")
    return v


def run_ddm(cfg: RunConfig, st: Setup, threads: int, quiet: bool, device: int = 0) -> int:
    """run_ddm (cli.cpp:170-205)."""
    t0 = time.perf_counter()
    prob = st.problem
    with DdmEngine(prob, device=device) as eng:
        _announce(quiet, _describe(prob, eng.sigma0()))
        f = sample_source(st)
        stats = DdmStats()
        u = eng.solve_iterative(f, cfg.tol, cfg.max_steps, stats, cfg.check_every)
        for r in stats.history:
            _announce(quiet, "step %4d  relres %.3e" % (r.step, r.relres))
        ra = RunArtifacts(mode="ddm", prob=prob, sigma0=eng.sigma0(), threads=threads,
                          classes=eng.class_info(), n_ddm_iter=stats.steps,
                          sweep_len=prob.n1 + prob.n2, relres=stats.relres,
                          converged=stats.converged, factor_ms=eng.factor_ms(),
                          solve_ms=stats.sweep_ms)
    ra.total_ms = (time.perf_counter() - t0) * 1e3
    write_field_artifacts(cfg, prob, u)
    write_resid_csv(cfg.prefix + "_resid.csv", [(r.step, r.relres, r.wall_ms) for r in stats.history])
    write_stats(cfg.prefix + "_stats.txt", ra)
    _announce(quiet, "%s after %d steps (n_DDM_Solv %.2f), relres %.3e" % (
        "converged" if stats.converged else "NOT converged", stats.steps,
        stats.steps / ra.sweep_len, stats.relres))
    return 0 if stats.converged else 3


def run_fgmres(cfg: RunConfig, st: Setup, threads: int, quiet: bool, device: int = 0) -> int:
    """run_fgmres (cli.cpp:207-260): FGMRES(A = apply_global, M = K sweeps)."""
    t0 = time.perf_counter()
    prob = st.problem
    K = cfg.precond_k if cfg.precond_k > 0 else prob.n1 + prob.n2
    with DdmEngine(prob, device=device) as eng:
        _announce(quiet, _describe(prob, eng.sigma0()))
        f = sample_source(st)
        pstats = DdmStats()
        x, kr = eng.fgmres(f, FgmresOptions(cfg.krylov_tol, cfg.krylov_max_iter,
                                            cfg.krylov_restart), K, pstats)
        ra = RunArtifacts(mode="fgmres", prob=prob, sigma0=eng.sigma0(), threads=threads,
                          classes=eng.class_info(), sweep_len=prob.n1 + prob.n2,
                          n_gmres_iter=kr.iters, precond_k=K, relres=kr.relres,
                          true_relres=kr.true_relres, converged=kr.converged,
                          factor_ms=eng.factor_ms(), solve_ms=pstats.sweep_ms)
    ra.total_ms = (time.perf_counter() - t0) * 1e3
    per_iter = kr.wall_ms / kr.iters if kr.iters else 0.0
    hist = [(i + 1, rel, per_iter) for i, rel in enumerate(kr.history)]
    write_field_artifacts(cfg, prob, x)
    write_resid_csv(cfg.prefix + "_resid.csv", hist)
    write_stats(cfg.prefix + "_stats.txt", ra)
    _announce(quiet, "%s in %d iterations (K=%d, n_Local_Solv %d), relres %.3e / true %.3e" % (
        "converged" if kr.converged else "NOT converged", kr.iters, K, kr.iters * K,
        kr.relres, kr.true_relres))
    return 0 if kr.converged else 3


def run_render(pos: Sequence[str], quiet: bool) -> int:
    """run_render (cli.cpp:420-427)."""
    if len(pos) != 2:
        raise ConfigError("render needs <dump> and <out.ppm>")
    nx, ny, _, _, _, data = read_field_dump(pos[0])
    write_ppm_real(pos[1], nx, ny, data, 0.0)
    _announce(quiet, "wrote " + pos[1])
    return 0


def _parse_args(argv: Sequence[str]):
    """parse_args (cli.cpp:37-60)."""
    cmd, pos, overrides, quiet, help_ = "", [], [], False, False
    i = 0
    while i < len(argv):
        s = argv[i]
        if s in ("-h", "--help"):
            help_ = True
        elif s == "--quiet":
            quiet = True
        elif s == "--override":
            if i + 1 >= len(argv):
                raise ConfigError("--override needs key=value")
            i += 1
            overrides.append(argv[i])
        elif s.startswith("--override="):
            overrides.append(s[len("--override="):])
        elif s and s[0] == "-":
            raise ConfigError("unknown option: " + s)
        elif not cmd:
            cmd = s
        else:
            pos.append(s)
        i += 1
    return cmd, pos, overrides, quiet, help_


def _dispatch(argv: Sequence[str]) -> int:
    """dispatch (cli.cpp:429-451)."""
    cmd, pos, overrides, quiet, help_ = _parse_args(argv)
    if help_ or not cmd:
        sys.stdout.write(USAGE)
        return 0 if help_ else 2
    if cmd == "render":
        return run_render(pos, quiet)
    if cmd not in ("solve", "direct", "convergence"):
        raise ConfigError("unknown command: " + cmd)
    if len(pos) != 1:
        raise ConfigError(cmd + " needs exactly one config file argument")
    cfg = parse_config_file(pos[0], overrides)
    threads = env_threads(cfg.threads)
    st = make_setup(cfg)
    mode = "direct" if cmd == "direct" else cfg.mode
    if cmd == "convergence" or mode == "direct":
        raise ConfigError(f"'{cmd if cmd != 'solve' else 'solver.mode = direct'}' factors the "
                          "global system on the host; not provided by the GPU engine")
    if mode == "ddm":
        return run_ddm(cfg, st, threads, quiet)
    return run_fgmres(cfg, st, threads, quiet)


def main(argv: Optional[Sequence[str]] = None) -> int:
    """run_cli (cli.cpp:453-469): exit codes 0 / 2 config / 3 solver / 4 io / 1 other."""
    argv = list(sys.argv[1:] if argv is None else argv)
    try:
        return _dispatch(argv)
    except ConfigError as e:
        sys.stderr.write(f"config error: {e}\n")
        return 2
    except SolveError as e:
        sys.stderr.write(f"solver error: {e}\n")
        return 3
    except IoError as e:
        sys.stderr.write(f"io error: {e}\n")
        return 4
    except (HddmError, Exception) as e:  # noqa: BLE001 -- mirrors catch(std::exception)
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
