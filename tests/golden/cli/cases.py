"""CLI parity cases: (name, config text without output.prefix, extra CLI args).

The first is the reference's own CLI test config (proj/tests/test_cli.cpp:33-47)."""
BASE = ("freq = 4\ngrid.ppw = 10\npart.n1 = 2\npart.n2 = 2\npml.n_overlap = 4\n"
        "pml.n_ramp = 8\nsolver.tol = 1e-8\nsolver.max_steps = 40\nthreads = 1\n")

CASES = [
    ("ddm_basic", BASE, []),
    ("fgmres_basic", BASE, ["--override", "solver.mode=fgmres"]),
    ("ddm_stall", BASE + "solver.max_steps = 1\n", []),
    ("layered_point", "freq = 3\ngrid.ppw = 12\npart.n1 = 3\npart.n2 = 2\n"
     "pml.n_overlap = 4\npml.n_ramp = 8\nmedium.type = layered\n"
     "medium.layers = 1.0, 1.5, 2.0\nsource.type = point\nsource.x = 0.3\nsource.y = 0.7\n"
     "solver.mode = fgmres\nkrylov.tol = 1e-9\nkrylov.restart = 10\nprecond.k = 3\n", []),
    ("ladder_h", "freq = 2.5\ngrid.h = 0.02\npart.n1 = 2\npart.n2 = 2\n"
     "domain.y1 = 0.9\npml.n_overlap = 3\npml.n_ramp = 6\nmedium.type = layered\n"
     "solver.tol = 1e-9\nsolver.max_steps = 30\nsolver.check_every = 2\n", []),
]
