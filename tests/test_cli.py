"""CLI parity on the host side (no GPU): the reference's test_cli.cpp /
test_config_io.cpp assertions re-expressed, and config / setup / source /
artifact writers compared with the UNMODIFIED reference (oracle/_ref, through
oracle/ref_capi.cpp)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1807_04180_b200 import cli
from paper_1807_04180_b200.engine import ConfigError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libhelmddm_ref.so")

BASE = ("freq = 4\ngrid.ppw = 10\npart.n1 = 2\npart.n2 = 2\npml.n_overlap = 4\n"
        "pml.n_ramp = 8\nsolver.tol = 1e-8\nsolver.max_steps = 40\nthreads = 1\n")


class _Setup(C.Structure):
    _fields_ = [("mx", C.c_int), ("my", C.c_int), ("n1", C.c_int), ("n2", C.c_int),
                ("n_overlap", C.c_int), ("n_ramp", C.c_int), ("h", C.c_double),
                ("x0", C.c_double), ("y0", C.c_double), ("omega", C.c_double),
                ("medium_kind", C.c_int), ("velocity", C.c_double), ("n_layers", C.c_int),
                ("layer_ylo", C.c_double * 64), ("layer_yhi", C.c_double * 64),
                ("layer_c", C.c_double * 64), ("source_kind", C.c_int),
                ("source_x", C.c_double), ("source_y", C.c_double), ("k_source", C.c_double),
                ("c_sigma", C.c_double), ("sigma0", C.c_double), ("mode", C.c_int),
                ("tol", C.c_double), ("krylov_tol", C.c_double), ("max_steps", C.c_int),
                ("check_every", C.c_int), ("precond_k", C.c_int), ("krylov_max_iter", C.c_int),
                ("krylov_restart", C.c_int), ("threads", C.c_int)]


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF_SO):
        pytest.skip("reference build oracle/_ref/libhelmddm_ref.so absent (make -C oracle ref)")
    return C.CDLL(REF_SO)


def ref_setup(lib, text, overrides=()):
    o = _Setup()
    err = C.create_string_buffer(512)
    rc = lib.ref_setup(text.encode(), "\n".join(overrides).encode(), C.byref(o), err, 512)
    return rc, o, err.value.decode()


SETUP_CASES = [
    BASE,
    BASE + "solver.mode = fgmres\n",
    "freq = 3\ngrid.ppw = 12\npart.n1 = 3\npart.n2 = 2\nmedium.type = layered\n"
    "medium.layers = 1.0, 1.5, 2.0\nsource.type = point\nsource.x = 0.3\nsource.y = 0.7\n",
    "freq = 2.5\ngrid.h = 0.02\npart.n1 = 2\npart.n2 = 2\ndomain.y1 = 0.9\nmedium.type = layered\n",
    "freq = 7\ngrid.ppw = 9.5\npart.n1 = 5\npart.n2 = 3\ndomain.x0 = -0.5\ndomain.x1 = 1.25\n"
    "domain.y0 = 0.2\ndomain.y1 = 1.9\nmedium.velocity = 1.7   # comment\npml.sigma0 = 12.5\n",
    "freq = 4\ngrid.ppw = 10\nmedium.type = layered\npart.n1 = 4\npart.n2 = 3\n"
    "domain.y1 = 1.37\n",
]


@pytest.mark.parametrize("text", SETUP_CASES)
def test_setup_matches_reference(ref, text):
    rc, o, err = ref_setup(ref, text)
    assert rc == 0, err
    st = cli.make_setup(cli.parse_config_text(text))
    p = st.problem
    assert (p.mx, p.my, p.n1, p.n2, p.n_overlap, p.n_ramp) == (o.mx, o.my, o.n1, o.n2,
                                                               o.n_overlap, o.n_ramp)
    assert p.h == o.h and p.x0 == o.x0 and p.y0 == o.y0 and p.omega == o.omega
    assert (p.medium_kind == 1) == (o.medium_kind == 1)
    if o.medium_kind == 1:
        assert [tuple(l) for l in p.layers] == [(o.layer_ylo[i], o.layer_yhi[i], o.layer_c[i])
                                               for i in range(o.n_layers)]
    else:
        assert p.velocity == o.velocity
    assert (st.source_kind == "point") == (o.source_kind == 1)
    assert st.source_x == o.source_x and st.source_y == o.source_y
    assert st.k_source == o.k_source
    assert p.c_sigma == o.c_sigma and p.sigma0 == o.sigma0


BAD_CASES = [
    "freq = 4\ngrid.ppw = 10\nwhat = 1\n",               # unknown key
    "grid.ppw = 10\n",                                   # freq missing
    "freq = 4\n",                                        # no spacing
    "freq = 4\ngrid.ppw = 10\ngrid.h = 0.1\n",           # both spacings
    "freq = 4\ngrid.ppw = 10\npart.n1 = 0\n",
    "freq = 4\ngrid.ppw = 10\npart.n1 = 1.5\n",          # not an integer
    "freq = 4x\ngrid.ppw = 10\n",                        # trailing garbage
    "freq = 4\ngrid.ppw = 10\nmedium.type = lens\n",
    "freq = 4\ngrid.ppw = 10\nsource.type = plane\n",
    "freq = 4\ngrid.ppw = 10\nsolver.mode = cg\n",
    "freq = 4\ngrid.ppw = 10\nmedium.layers = 1, -2\n",
    "freq = 4\ngrid.ppw = 10\nno equals sign\n",
    "freq = 4\ngrid.ppw = 10\n = 3\n",
    "freq = 4\ngrid.ppw = 10\noutput.prefix =\n",
    "freq = 4\ngrid.ppw = 10\nsolver.check_every = 0\n",
    "freq = 4\ngrid.ppw = 10\nconv.ref = exact\n",
]


@pytest.mark.parametrize("text", BAD_CASES)
def test_config_errors_match_reference(ref, text):
    rc, _, err = ref_setup(ref, text)
    assert rc == 2
    with pytest.raises(ConfigError) as e:
        cli.parse_config_text(text)
    assert str(e.value) == err


def test_overrides_match_reference(ref):
    ov = ["solver.mode=fgmres", "part.n1 = 4", "medium.type=layered", "source.y=0.25"]
    rc, o, err = ref_setup(ref, BASE, ov)
    assert rc == 0, err
    c = cli.parse_config_text(BASE, ov)
    st = cli.make_setup(c)
    assert c.mode == "fgmres" and o.mode == 1
    assert st.problem.n1 == o.n1 == 4
    assert st.source_y == o.source_y == 0.25 and st.source_x == o.source_x == 0.0
    with pytest.raises(ConfigError):
        cli.parse_config_text(BASE, ["novalue"])


@pytest.mark.parametrize("text", SETUP_CASES[:3])
def test_source_matches_reference(ref, text):
    st = cli.make_setup(cli.parse_config_text(text))
    f = cli.sample_source(st)
    g = np.zeros(f.size * 2, np.float64)
    assert ref.ref_sample_source(text.encode(), g.ctypes.data_as(C.POINTER(C.c_double))) == 0
    g = g.view(np.complex128)
    # numpy's exp may differ from glibc's by an ulp
    np.testing.assert_allclose(f, g, rtol=2e-15, atol=0)


REF_EXE = os.path.join(ROOT, "oracle", "_ref", "helmddm")
GOLD = os.path.join(ROOT, "tests", "golden", "cli")


def test_writers_match_reference_bytes(tmp_path):
    """Our HDMF dump read by the reference `helmddm render` (io.cpp:46-69) gives
    the reference image (io.cpp:71-99) byte for byte equal to ours."""
    if not os.path.exists(REF_EXE):
        pytest.skip("reference CLI oracle/_ref/helmddm absent (make -C oracle ref-cli)")
    import subprocess
    rng = np.random.default_rng(5)
    nx, ny = 37, 23
    data = (rng.standard_normal(nx * ny) + 1j * rng.standard_normal(nx * ny)).astype(np.complex128)
    data[:5] = [0, 1, -1, 0.5, -0.25]
    dump = tmp_path / "d.hdmf"
    cli.write_field_dump(str(dump), nx, ny, -0.3, 0.125, 1 / 64, data)
    ours, theirs = tmp_path / "ours.ppm", tmp_path / "ref.ppm"
    cli.write_ppm_real(str(ours), nx, ny, data, 0.0)
    r = subprocess.run([REF_EXE, "render", str(dump), str(theirs), "--quiet"], capture_output=True)
    assert r.returncode == 0, r.stderr
    assert ours.read_bytes() == theirs.read_bytes()
    assert cli.main(["render", str(dump), str(tmp_path / "again.ppm"), "--quiet"]) == 0
    assert (tmp_path / "again.ppm").read_bytes() == theirs.read_bytes()
    nx2, ny2, x0, y0, h, d2 = cli.read_field_dump(str(dump))
    assert (nx2, ny2, x0, y0, h) == (nx, ny, -0.3, 0.125, 1 / 64)
    assert np.array_equal(d2, data)


@pytest.mark.parametrize("name", ["ddm_basic", "fgmres_basic", "layered_point"])
def test_resid_csv_format_matches_reference(tmp_path, name):
    g = np.load(os.path.join(GOLD, name + ".npz"))
    text = str(g["resid"])
    rows = [l.split(",") for l in text.strip().split("\n")[1:]]
    hist = [(int(a), float(b), float(c)) for a, b, c in rows]
    out = tmp_path / "r.csv"
    cli.write_resid_csv(str(out), hist)
    assert out.read_text() == text


def test_dump_reader_rejects_bad_files(tmp_path):
    bad = tmp_path / "x.hdmf"
    bad.write_bytes(b"NOPE" + bytes(40))
    with pytest.raises(cli.IoError):
        cli.read_field_dump(str(bad))
    good = tmp_path / "g.hdmf"
    cli.write_field_dump(str(good), 2, 2, 0, 0, 1, np.zeros(4, np.complex128))
    good.write_bytes(good.read_bytes() + b"\0")
    with pytest.raises(cli.IoError, match="trailing"):
        cli.read_field_dump(str(good))
    good.write_bytes(good.read_bytes()[:-20])
    with pytest.raises(cli.IoError, match="truncated"):
        cli.read_field_dump(str(good))


def test_exit_codes_without_a_solve(tmp_path, capsys):
    """test_cli.cpp:64-70 and :148-157 (the parts that need no solve)."""
    assert cli.main([]) == 2
    assert cli.main(["--help"]) == 0
    assert cli.main(["frobnicate", "x.cfg"]) == 2
    assert cli.main(["--bad-flag"]) == 2
    assert cli.main(["solve"]) == 2
    assert cli.main(["solve", str(tmp_path / "missing.cfg")]) == 4
    bad = tmp_path / "bad.cfg"
    bad.write_text("freq = 4\ngrid.ppw = 10\nwhat = 1\n")
    assert cli.main(["solve", str(bad)]) == 2
    assert cli.main(["render", str(tmp_path / "nothing.hdmf"), str(tmp_path / "x.ppm")]) == 4
    assert cli.main(["render", "only-one-arg"]) == 2
    good = tmp_path / "good.cfg"
    good.write_text(BASE)
    assert cli.main(["direct", str(good)]) == 2  # host global factorization: not on the GPU path
    os.environ["HELMDDM_THREADS"] = "abc"
    try:
        assert cli.main(["solve", str(good)]) == 2
    finally:
        del os.environ["HELMDDM_THREADS"]
    err = capsys.readouterr().err
    assert "config error: unknown config key: what" in err
    assert "io error: cannot open config file" in err


def test_stats_format(tmp_path):
    from paper_1807_04180_b200.problems import Problem
    p = Problem(name="t", mx=40, my=40, h=0.025, n1=2, n2=2, n_overlap=4, n_ramp=8, omega=8.0)
    ra = cli.RunArtifacts(mode="fgmres", prob=p, sigma0=14.921, threads=3,
                          classes=[{"backend": "ldlt"}] * 4, sweep_len=4, n_gmres_iter=5,
                          precond_k=4, relres=3.1e-9, true_relres=2.9e-9, converged=True,
                          factor_ms=1.25, solve_ms=10.0, total_ms=20.04)
    path = tmp_path / "s.txt"
    cli.write_stats(str(path), ra)
    assert path.read_text() == (
        "mode = fgmres\ngrid.cells = 40 x 40\ngrid.h = 2.500000000e-02\npartition = 2 x 2\n"
        "pml.n_ramp = 8\npml.n_overlap = 4\npml.sigma0 = 1.492100000e+01\nthreads = 3\n"
        "factor.classes = 4\nfactor.backend.ldlt = 4\nfactor.backend.lu = 0\nn_DDM_Iter = 0\n"
        "n_DDM_Solv = 0.00\nn_GMRES_Iter = 5\nn_Local_Solv = 20\nprecond.k = 4\n"
        "relres = 3.100000e-09\ntrue_relres = 2.900000e-09\nconverged = yes\n"
        "factor_ms = 1.2\nsolve_ms = 10.0\ntotal_ms = 20.0\n")
