"""CLI end to end on the GPU engine vs the reference command line's recorded
artifacts (tests/golden/cli, made by tests/golden/make_golden_cli.py from the
UNMODIFIED reference `helmddm`): exit code, field dump, stats keys, residual
history, image; plus the reference CLI test's own assertions
(proj/tests/test_cli.cpp:72-146)."""
import os

import numpy as np
import pytest

from paper_1807_04180_b200 import cli

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "cli")

import sys  # noqa: E402

sys.path.insert(0, GOLD)
from cases import CASES  # noqa: E402

TIMING = ("factor_ms", "solve_ms", "total_ms")


def _stats(text):
    out = {}
    for line in text.strip().split("\n"):
        k, v = line.split(" = ", 1)
        out[k] = v
    return out


def _run(tmp_path, name, text, args):
    prefix = str(tmp_path / name)
    cfg = tmp_path / (name + ".cfg")
    cfg.write_text(text + f"output.prefix = {prefix}\n")
    rc = cli.main(["solve", str(cfg), "--quiet"] + list(args))
    return rc, prefix


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_cli_matches_reference_run(tmp_path, case):
    name, text, args = case
    g = np.load(os.path.join(GOLD, name + ".npz"))
    rc, prefix = _run(tmp_path, name, text, args)
    assert rc == int(g["rc"])
    for suffix in ("_field.hdmf", "_real.ppm", "_resid.csv", "_stats.txt"):
        assert os.path.exists(prefix + suffix)
    nx, ny, x0, y0, h, u = cli.read_field_dump(prefix + "_field.hdmf")
    assert (nx, ny) == (int(g["nx"]), int(g["ny"]))
    assert (x0, y0, h) == (float(g["x0"]), float(g["y0"]), float(g["h"]))
    ref = g["field"]
    rel = np.linalg.norm(u - ref) / np.linalg.norm(ref)
    assert rel <= 1e-8, rel
    ours, theirs = _stats(open(prefix + "_stats.txt").read()), _stats(str(g["stats"]))
    assert ours.keys() == theirs.keys()
    for k in ours:
        if k in TIMING:
            continue
        if k in ("relres", "true_relres"):
            a, b = float(ours[k]), float(theirs[k])
            assert abs(a - b) <= 1e-3 * abs(b) + 1e-12, (k, a, b)
        else:
            assert ours[k] == theirs[k], (k, ours[k], theirs[k])
    rows = lambda t: [l.split(",") for l in t.strip().split("\n")[1:]]  # noqa: E731
    ro, rt = rows(open(prefix + "_resid.csv").read()), rows(str(g["resid"]))
    assert [r[0] for r in ro] == [r[0] for r in rt]
    for a, b in zip(ro, rt):
        assert abs(float(a[1]) - float(b[1])) <= 1e-3 * float(b[1]) + 1e-12


def test_reference_cli_assertions(tmp_path):
    """test_cli.cpp:72-146: artifacts, header, classes, the fgmres solve-count
    identity, render byte for byte."""
    base = CASES[0][1]
    rc, prefix = _run(tmp_path, "run1", base, [])
    assert rc == 0
    nx, ny, *_ = cli.read_field_dump(prefix + "_field.hdmf")
    assert nx == 40 + 2 * 12 + 1 and ny == nx
    stats = open(prefix + "_stats.txt").read()
    assert "mode = ddm" in stats and "converged = yes" in stats
    assert "factor.classes = 4" in stats
    assert open(prefix + "_resid.csv").readline().strip() == "step,relres,wall_ms"
    rc, kp = _run(tmp_path, "kry1", base, ["--override", "solver.mode=fgmres"])
    assert rc == 0
    s = _stats(open(kp + "_stats.txt").read())
    assert s["mode"] == "fgmres" and int(s["precond.k"]) == 4
    assert int(s["n_Local_Solv"]) == int(s["n_GMRES_Iter"]) * 4 and int(s["n_GMRES_Iter"]) >= 1
    assert "true_relres" in s
    out = str(tmp_path / "rerender.ppm")
    assert cli.main(["render", prefix + "_field.hdmf", out, "--quiet"]) == 0
    assert open(out, "rb").read() == open(prefix + "_real.ppm", "rb").read()
    # HELMDDM_THREADS is reported and changes nothing
    os.environ["HELMDDM_THREADS"] = "3"
    try:
        rc, p3 = _run(tmp_path, "thr3", base, [])
    finally:
        del os.environ["HELMDDM_THREADS"]
    assert rc == 0 and "threads = 3" in open(p3 + "_stats.txt").read()
    a = cli.read_field_dump(prefix + "_field.hdmf")[-1]
    b = cli.read_field_dump(p3 + "_field.hdmf")[-1]
    assert np.array_equal(a, b)
