"""Host input generator: RNG known answers, config geometry (CPU)."""
import math

import numpy as np

from paper_1807_04180_b200.problems import MT19937_64, config, random_layers, small


def test_mt19937_64_known_answer():
    # C++11 [rand.predef]: the 10000th output of a default-constructed mt19937_64
    r = MT19937_64()
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042


def test_mt19937_64_seed0_prefix():
    r = MT19937_64(0)
    assert [r.next_u64() for _ in range(3)] == [2947667278772165694, 18301848765998365067,
                                                  729919693006235833]


def test_random_layers_cfg4():
    lay = random_layers(20, 0)
    assert len(lay) == 20
    cuts = [l[0] for l in lay[1:]]
    assert cuts == sorted(cuts) and lay[0][0] == 0.0 and lay[-1][1] == 1.0
    assert all(1.0 <= c <= 3.0 for *_, c in lay)
    # c_min = 1.0399, omega = 2 pi c_min 2048 / 8 ~ 532.4 pi
    p = config(4)
    assert abs(p.c_min() - 1.0399) < 1e-4
    assert abs(p.omega / math.pi - 532.41) < 1e-2


def test_config_geometry():
    # window and global sizes
    assert config(1).window == (105, 105) and config(1).n_global == 88209
    assert config(2).window == (193, 193) and config(2).n_global == 1185921
    assert config(4).window == (193, 193) and config(4).n_global == 4464769
    assert config(4).nsub == 256 and config(4).k_steps == 32
    assert config(2).k_steps == 16


def test_sources():
    p = config(1)
    f = p.source_f()
    assert f.shape == (p.n_global,) and f.dtype == np.complex128
    assert abs(f.max() - 1.0) < 1e-12 and np.all(f.imag == 0)
    q = small(source=("point", 0.3, 0.6))
    g = q.source_f()
    assert np.count_nonzero(g) == 1 and g.max() == 1.0 / q.h ** 2
