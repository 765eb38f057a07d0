"""C-ABI boundary (CPU): the library loads, exports every symbol include/hddm.h
declares, runs its host-only symbolic analysis, and refuses to run without a
GPU (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1807_04180_b200 import engine


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "hddm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hddm_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(engine.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_nd_order_matches_oracle_and_reference_rules():
    import pyoracle
    for nx, ny in ((45, 45), (105, 105), (57, 40), (8, 9)):
        a = engine.nd_order(nx, ny)
        b = pyoracle.nd_order(nx, ny)
        assert np.array_equal(a, b)
        assert np.array_equal(np.sort(a), np.arange(nx * ny))  # a permutation
        # ring first (sparse.cpp:42-57)
        nring = 2 * nx + 2 * (ny - 2)
        ring = {q * nx + p for q in range(ny) for p in range(nx)
                if p in (0, nx - 1) or q in (0, ny - 1)}
        assert set(a[:nring].tolist()) == ring


@pytest.mark.parametrize("w,nnz", [(45, 37712), (101, 284272), (105, 316428), (193, 1287272)])
def test_symbolic_nnz_equals_reference_factor_nonzeros(w, nnz):
    # reference factor_nonzeros() (sparse.cpp:238-240) recorded by the goldens /
    # the survey probes: the engine's profile storage holds exactly nnz(L)
    st = engine.symbolic_stats(w, w)
    assert st["nnz_ref"] == nnz
    assert st["stored"] == nnz - w * w


def test_symbolic_matches_golden_class_nnz():
    from conftest import golden_cases, golden
    for name, prob, _ in golden_cases():
        g = golden(name)
        nx, ny = prob.window
        assert engine.symbolic_stats(nx, ny)["nnz_ref"] == int(g["factor_nnz"][0])


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1807_04180_b200.problems import small
    with pytest.raises(engine.HddmError, match="CUDA"):
        engine.DdmEngine(small())


def test_config_errors_map_to_config_error():
    # partition check (partition.cpp:15-28) runs before any device work
    import torch
    from paper_1807_04180_b200.problems import small
    bad = small(41, 2, 2)  # 41 cells do not split in two
    with pytest.raises(engine.ConfigError, match="divide evenly"):
        engine.DdmEngine(bad)


# ---------------------------------------------------------------- 3-D path (hddm3.h)
def declared_symbols3():
    txt = open(os.path.join(ROOT, "include", "hddm3.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hddm3_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_3d_symbol():
    lib = ctypes.CDLL(engine.LIB_PATH)
    syms = declared_symbols3()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


@pytest.mark.parametrize("dims", [(11, 9, 13), (19, 19, 19), (25, 17, 21)])
def test_3d_order_and_nnz_match_restatement(dims):
    import pyoracle
    from paper_1807_04180_b200 import engine3
    assert np.array_equal(engine3.nd_order3(*dims), pyoracle.nd_order3(*dims))
    st = engine3.symbolic_stats3(*dims)
    # the restatement's up-looking LDL^T of the same order: exact nnz(L) + n
    if dims == (19, 19, 19):
        from paper_1807_04180_b200.problems import small3
        o = pyoracle.Oracle3Engine(small3())
        assert st["nnz_ref"] == o.class_info()[0]["factor_nnz"]
    assert st["stored"] >= st["nnz_ref"]  # dense supernode blocks hold every entry of L


def test_3d_config5_symbolic_footprint():
    from paper_1807_04180_b200 import engine3
    from paper_1807_04180_b200.problems import config5
    st = engine3.symbolic_stats3(*config5().window)
    # 57^3 windows: nnz(L) + n = 83,587,619; the dense supernode storage 3.3 % more
    assert st["nnz_ref"] == 83587619
    assert st["stored"] < 1.04 * st["nnz_ref"]
    assert 8 * 16 * st["stored"] < 12e9  # eight classes of factors: 11.1 GB of 180 GB


def test_3d_config_errors_map_to_config_error():
    from paper_1807_04180_b200 import engine3
    from paper_1807_04180_b200.problems import small3
    with pytest.raises(engine.ConfigError, match="divide evenly"):
        engine3.DdmEngine3(small3(m=17, n=2))
