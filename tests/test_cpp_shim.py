"""The header-only C++ shim (include/helmddm_b200/ddm.hpp) compiles against the
C-ABI (CPU) and runs the reference-style scenarios on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
LIBDIR = os.path.join(ROOT, "paper_1807_04180_b200")


def build(tmp_path):
    exe = str(tmp_path / "test_shim")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lhddm", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_shim_runs_reference_scenarios(tmp_path):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim ok" in out.stdout


def test_host_fgmres_dense_system(tmp_path):
    """The shim's fgmres(n, A, M, b, x, opt) over LinearOp callbacks (CPU)."""
    exe = str(tmp_path / "test_fgmres_host")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_fgmres_host.cpp"), "-o", exe],
                   check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "host fgmres ok" in out.stdout
