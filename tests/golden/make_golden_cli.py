"""Record the UNMODIFIED reference CLI's artifacts for the CLI parity tests.

Run in the build container (needs `make -C oracle ref-cli`):
    python tests/golden/make_golden_cli.py
For every case in tests/golden/cli/cases.py the reference command line
(oracle/_ref/helmddm = proj/tools/helmddm_main.cpp -> run_cli) solves the
config on the CPU; the field dump is stored as complex128 in
tests/golden/cli/<name>.npz together with the stats text and the residual CSV.
The GPU box has no /root/reference: tests/test_gpu_cli.py compares the B200
CLI's artifacts with these files.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(HERE, "cli"))

from cases import CASES  # noqa: E402


def ref_cli(exe, args):
    env = dict(os.environ, HELMDDM_THREADS="1")
    return subprocess.run([exe] + list(args), env=env, capture_output=True).returncode


def main():
    exe = os.path.join(ROOT, "oracle", "_ref", "helmddm")
    sys.path.insert(0, ROOT)
    from paper_1807_04180_b200.cli import read_field_dump
    with tempfile.TemporaryDirectory() as d:
        for name, text, args in CASES:
            prefix = os.path.join(d, name)
            cfg = os.path.join(d, name + ".cfg")
            with open(cfg, "w") as f:
                f.write(text + f"output.prefix = {prefix}\n")
            rc = ref_cli(lib, ["solve", cfg, "--quiet"] + list(args))
            nx, ny, x0, y0, h, data = read_field_dump(prefix + "_field.hdmf")
            stats = open(prefix + "_stats.txt").read()
            resid = open(prefix + "_resid.csv").read()
            np.savez_compressed(os.path.join(HERE, "cli", name + ".npz"), rc=rc, nx=nx, ny=ny,
                                x0=x0, y0=y0, h=h, field=data, stats=stats, resid=resid)
            print(name, "rc", rc, "field", nx, ny)


if __name__ == "__main__":
    main()
