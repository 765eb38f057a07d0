"""Problem descriptions and the shared host input generator.

One ``Problem`` carries what the reference's ``DdmConfig`` carries
(``GridSpec`` proj/include/helmddm/partition.hpp:13-31, ``MediumModel``
proj/include/helmddm/medium.hpp:17-29, ``c_sigma``/``sigma0``
proj/include/helmddm/ddm.hpp:15-22) plus the run recipe of a BASELINE.json
config. Sources and media are generated ONCE on the host and handed to every
implementation (CUDA engine, C restatement, reference) so all of them consume
byte-identical inputs.

Stand-ins for BASELINE.json configs (seeded synthetic inputs, no dataset):

=====  ===========================================================  =========
cfg    geometry / medium / source                                   run
=====  ===========================================================  =========
1      256^2, 4x4, ov 4, PML 16, c=1, w=40pi, Gaussian s=0.01 (.5,.5)  10 standalone steps
2      1024^2, 8x8, ov 8, PML 24, c=1, w=160pi, s=0.005 centred       FGMRES(30)+DDM(K=16)
3      1024^2, 8x8, lens c=1-0.4exp(-r^2/0.05), w=120pi, s=.005@(.25,.25)  FGMRES(30)+DDM(K=16)
4      2048^2, 16x16, ov 8, PML 24, 20 random layers (mt19937_64 seed 0),
       w = 2pi c_min 2048/8, s=0.003 @ (0.5, 0.1)                   FGMRES(30)+DDM(K=32)
5      3-D 64^3, 2x2x2, ov 4, PML 8, c=1, w=16pi, 3-D Gaussian
       s=0.02 at the cube centre (``Problem3``; no reference)       FGMRES(30)+DDM(K=6)
=====  ===========================================================  =========

``h = 1/mx`` for cfg 1: "256x256 interior, h=1/257" cannot be split four ways;
the reference's own snapping (proj/src/config.cpp:206-210) maps it to mx=256
(SURVEY.md 8(d) note).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import List, Optional, Tuple

import numpy as np

MEDIUM_CONSTANT, MEDIUM_LAYERED, MEDIUM_LENS = 0, 1, 2


class MT19937_64:
    """64-bit Mersenne Twister (the published MT19937-64 recurrence), used to
    draw config 4's layer cuts and velocities exactly as ``std::mt19937_64(0)``
    would."""

    _N, _M = 312, 156
    _A = 0xB5026F5AA96619E9
    _UM, _LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
    _MASK = (1 << 64) - 1

    def __init__(self, seed: int = 5489):
        self.mt = [0] * self._N
        self.mt[0] = seed & self._MASK
        for i in range(1, self._N):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & self._MASK
        self.idx = self._N

    def _twist(self):
        mt = self.mt
        for i in range(self._N):
            x = (mt[i] & self._UM) | (mt[(i + 1) % self._N] & self._LM)
            xa = x >> 1
            if x & 1:
                xa ^= self._A
            mt[i] = mt[(i + self._M) % self._N] ^ xa
        self.idx = 0

    def next_u64(self) -> int:
        if self.idx >= self._N:
            self._twist()
        x = self.mt[self.idx]
        self.idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & self._MASK

    def uniform01(self) -> float:
        """u = (x >> 11) * 2^-53."""
        return float(self.next_u64() >> 11) * 2.0 ** -53


@dataclass
class Problem:
    name: str
    mx: int
    n1: int
    n2: int
    n_overlap: int
    n_ramp: int
    omega: float
    my: int = 0
    h: float = 0.0
    x0: float = 0.0
    y0: float = 0.0
    medium_kind: int = MEDIUM_CONSTANT
    velocity: float = 1.0
    layers: List[Tuple[float, float, float]] = field(default_factory=list)
    lens: Tuple[float, float, float, float] = (0.0, 0.0, 0.0, 1.0)  # amp, xc, yc, w
    c_sigma: float = 25.0
    sigma0: float = 0.0
    # source: ("gaussian", xc, yc, sigma) -> exp(-r^2 / (2 sigma^2));
    #         ("point", x, y) -> 1/h^2 at the nearest node (medium.cpp:55-60)
    source: Tuple = ("gaussian", 0.5, 0.5, 0.01)
    mode: str = "standalone"  # standalone | fgmres
    steps: int = 10           # standalone max_steps
    tol: float = 0.0
    K: int = 0                # 0 -> n1 + n2 (proj/src/cli.cpp:217)
    restart: int = 30
    max_iters: int = 200

    def __post_init__(self):
        if self.my == 0:
            self.my = self.mx
        if self.h == 0.0:
            self.h = 1.0 / self.mx

    # GridSpec helpers (partition.hpp:20-31)
    @property
    def n_ext(self) -> int:
        return self.n_overlap + self.n_ramp

    @property
    def gnx(self) -> int:
        return self.mx + 2 * self.n_ext + 1

    @property
    def gny(self) -> int:
        return self.my + 2 * self.n_ext + 1

    @property
    def n_global(self) -> int:
        return self.gnx * self.gny

    @property
    def window(self) -> Tuple[int, int]:
        return (self.mx // self.n1 + 2 * self.n_ext + 1,
                self.my // self.n2 + 2 * self.n_ext + 1)

    @property
    def nsub(self) -> int:
        return self.n1 * self.n2

    @property
    def k_steps(self) -> int:
        return self.K if self.K > 0 else self.n1 + self.n2

    def c_min(self) -> float:
        if self.medium_kind == MEDIUM_LAYERED:
            return min(c for _, _, c in self.layers)
        if self.medium_kind == MEDIUM_LENS:
            return self.velocity - self.lens[0]  # lens centre lies inside
        return self.velocity

    def lattice_xy(self):
        ox = self.x0 - self.n_ext * self.h
        oy = self.y0 - self.n_ext * self.h
        p = np.arange(self.gnx, dtype=np.float64)
        q = np.arange(self.gny, dtype=np.float64)
        return ox + p * self.h, oy + q * self.h

    def source_f(self) -> np.ndarray:
        """Global-window source, complex128, row-major x fastest (length n_global)."""
        xs, ys = self.lattice_xy()
        kind = self.source[0]
        if kind == "gaussian":
            _, xc, yc, sig = self.source
            dx2 = (xs - xc) ** 2
            dy2 = (ys - yc) ** 2
            f = np.exp(-(dy2[:, None] + dx2[None, :]) / (2.0 * sig * sig))
            return f.astype(np.complex128).ravel()
        if kind == "point":
            _, x, y = self.source
            ox = self.x0 - self.n_ext * self.h
            oy = self.y0 - self.n_ext * self.h
            p = int(math.ceil((x - ox) / self.h - 0.5))
            q = int(math.ceil((y - oy) / self.h - 0.5))
            f = np.zeros((self.gny, self.gnx), np.complex128)
            if 0 <= p < self.gnx and 0 <= q < self.gny:
                f[q, p] = 1.0 / (self.h * self.h)
            return f.ravel()
        raise ValueError(f"unknown source kind {kind!r}")

    def with_(self, **kw) -> "Problem":
        return replace(self, **kw)


def random_layers(n_layers: int = 20, seed: int = 0, c_lo: float = 1.0,
                  c_hi: float = 3.0) -> List[Tuple[float, float, float]]:
    """Config 4's medium: n_layers-1 interface depths ~U(0,1) sorted, drawn
    first, then n_layers velocities ~U[c_lo, c_hi]; band 0 at the bottom
    (y = depth, medium.hpp:21)."""
    rng = MT19937_64(seed)
    cuts = sorted(rng.uniform01() for _ in range(n_layers - 1))
    cs = [c_lo + (c_hi - c_lo) * rng.uniform01() for _ in range(n_layers)]
    edges = [0.0] + cuts + [1.0]
    return [(edges[i], edges[i + 1], cs[i]) for i in range(n_layers)]


def config(n: int) -> Problem:
    """BASELINE.json configs 1-4 (0-based index n-1)."""
    if n == 1:
        return Problem("cfg1_256_4x4_standalone", mx=256, n1=4, n2=4, n_overlap=4,
                       n_ramp=16, omega=40 * math.pi, source=("gaussian", 0.5, 0.5, 0.01),
                       mode="standalone", steps=10, tol=0.0)
    if n == 2:
        return Problem("cfg2_1024_8x8_fgmres", mx=1024, n1=8, n2=8, n_overlap=8,
                       n_ramp=24, omega=160 * math.pi,
                       source=("gaussian", 0.5, 0.5, 0.005), mode="fgmres",
                       tol=1e-6, K=16, restart=30, max_iters=200)
    if n == 3:
        return Problem("cfg3_1024_8x8_lens_fgmres", mx=1024, n1=8, n2=8, n_overlap=8,
                       n_ramp=24, omega=120 * math.pi, medium_kind=MEDIUM_LENS,
                       velocity=1.0, lens=(0.4, 0.5, 0.5, 0.05),
                       source=("gaussian", 0.25, 0.25, 0.005), mode="fgmres",
                       tol=1e-6, K=16, restart=30, max_iters=200)
    if n == 4:
        layers = random_layers(20, 0)
        cmin = min(c for _, _, c in layers)
        return Problem("cfg4_2048_16x16_layered_fgmres", mx=2048, n1=16, n2=16,
                       n_overlap=8, n_ramp=24, omega=2 * math.pi * cmin * 2048 / 8,
                       medium_kind=MEDIUM_LAYERED, layers=layers,
                       source=("gaussian", 0.5, 0.1, 0.003), mode="fgmres",
                       tol=1e-6, K=32, restart=30, max_iters=200)
    if n == 5:
        return config5()
    raise ValueError(f"config {n} not available (configs 1-5)")


def small(mx: int = 40, n1: int = 2, n2: int = 2, freq: float = 4.0, n_ov: int = 4,
          n_ramp: int = 8, source=("point", 0.3, 0.6), **kw) -> Problem:
    """The reference tests' ``make_cfg`` (proj/tests/test_ddm.cpp:15-30)."""
    return Problem(f"small_{mx}_{n1}x{n2}", mx=mx, n1=n1, n2=n2, n_overlap=n_ov,
                   n_ramp=n_ramp, omega=2 * math.pi * freq, source=source, **kw)


@dataclass
class Problem3:
    """A 3-D problem (BASELINE config 5): the 2-D ``Problem`` with a third axis
    and a constant medium. The reference has no 3-D code; the
    formulas are the generalization written out in oracle/hddm_oracle3.c."""
    name: str
    mx: int
    n1: int
    n2: int
    n3: int
    n_overlap: int
    n_ramp: int
    omega: float
    my: int = 0
    mz: int = 0
    h: float = 0.0
    x0: float = 0.0
    y0: float = 0.0
    z0: float = 0.0
    velocity: float = 1.0
    c_sigma: float = 25.0
    sigma0: float = 0.0
    source: Tuple = ("gaussian", 0.5, 0.5, 0.5, 0.02)  # exp(-r^2 / (2 sigma^2))
    mode: str = "fgmres"
    steps: int = 10
    tol: float = 1e-6
    K: int = 0                # 0 -> n1 + n2 + n3
    restart: int = 30
    max_iters: int = 200

    def __post_init__(self):
        if self.my == 0:
            self.my = self.mx
        if self.mz == 0:
            self.mz = self.mx
        if self.h == 0.0:
            self.h = 1.0 / self.mx

    @property
    def n_ext(self) -> int:
        return self.n_overlap + self.n_ramp

    @property
    def gdims(self) -> Tuple[int, int, int]:
        e = 2 * self.n_ext + 1
        return (self.mx + e, self.my + e, self.mz + e)

    @property
    def n_global(self) -> int:
        a, b, c = self.gdims
        return a * b * c

    @property
    def window(self) -> Tuple[int, int, int]:
        e = 2 * self.n_ext + 1
        return (self.mx // self.n1 + e, self.my // self.n2 + e, self.mz // self.n3 + e)

    @property
    def nsub(self) -> int:
        return self.n1 * self.n2 * self.n3

    @property
    def k_steps(self) -> int:
        return self.K if self.K > 0 else self.n1 + self.n2 + self.n3

    def source_f(self) -> np.ndarray:
        """Global-window source, complex128, x fastest then y then z."""
        gx, gy, gz = self.gdims
        e = self.n_ext * self.h
        xs = self.x0 - e + np.arange(gx) * self.h
        ys = self.y0 - e + np.arange(gy) * self.h
        zs = self.z0 - e + np.arange(gz) * self.h
        kind = self.source[0]
        if kind == "gaussian":
            _, xc, yc, zc, sig = self.source
            r2 = ((zs - zc) ** 2)[:, None, None] + ((ys - yc) ** 2)[None, :, None] + \
                ((xs - xc) ** 2)[None, None, :]
            return np.exp(-r2 / (2.0 * sig * sig)).astype(np.complex128).ravel()
        if kind == "point":
            _, x, y, z = self.source
            f = np.zeros((gz, gy, gx), np.complex128)
            idx = [int(math.ceil((v - (o - e)) / self.h - 0.5)) for v, o in
                   ((x, self.x0), (y, self.y0), (z, self.z0))]
            if 0 <= idx[0] < gx and 0 <= idx[1] < gy and 0 <= idx[2] < gz:
                f[idx[2], idx[1], idx[0]] = 1.0 / (self.h ** 3)
            return f.ravel()
        raise ValueError(f"unknown source kind {kind!r}")

    def with_(self, **kw) -> "Problem3":
        return replace(self, **kw)


def config5() -> Problem3:
    """BASELINE config 5: 64^3, 2x2x2, overlap 4, PML 8, c=1, w=16pi, 3-D
    Gaussian sigma=0.02 at the centre, FGMRES(30)+DDM(K=6) to 1e-6
    (SURVEY.md 8(d))."""
    return Problem3("cfg5_64cube_2x2x2_fgmres", mx=64, n1=2, n2=2, n3=2, n_overlap=4,
                    n_ramp=8, omega=16 * math.pi, source=("gaussian", 0.5, 0.5, 0.5, 0.02),
                    mode="fgmres", tol=1e-6, K=6, restart=30, max_iters=200)


def small3(m: int = 16, n: int = 2, freq: float = 3.0, n_ov: int = 2, n_ramp: int = 3,
           source=("gaussian", 0.45, 0.55, 0.5, 0.08), **kw) -> Problem3:
    """A small 3-D case the C restatement factors in well under a second."""
    return Problem3(f"small3_{m}_{n}", mx=m, n1=n, n2=n, n3=n, n_overlap=n_ov,
                    n_ramp=n_ramp, omega=2 * math.pi * freq, source=source, **kw)
