"""Golden bundles: run the REAL reference CLI (build container only).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_bundles.py

Writes under tests/golden/bundles/:
* phys/      `hsdla gen --seed 11 --atoms 4 --lsph 3 --lnonsph 2 --basis-factor 50
               --hpd-fraction 0.5` (physics coefficients, system.json, 2 HPD + 2 non-HPD atoms)
* phys_out/  `hsdla build phys` (H.hsm1, S.hsm1, report.json)
* rand/      `hsdla gen --seed 12 --atoms 2 --lsph 2 --lnonsph 1 --basis-factor 40
               --coeffs random` (no system.json)
* rand_out/  `hsdla build rand`
These pin `paper_1602_06589_b200.bundle.build_bundle` and the HSM1 reader/writer
(tests/test_bundle.py).
"""
from __future__ import annotations

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "bundles")
sys.path.insert(0, "/root/reference/pkg/src")

from hsdla.cli import main  # noqa: E402  (the reference)


def run(argv):
    rc = main(argv)
    if rc != 0:
        raise SystemExit(f"reference CLI failed ({rc}): {argv}")


if __name__ == "__main__":
    shutil.rmtree(OUT, ignore_errors=True)
    p = lambda name: os.path.join(OUT, name)  # noqa: E731
    run(["gen", "--seed", "11", "--atoms", "4", "--lsph", "3", "--lnonsph", "2",
         "--basis-factor", "50", "--hpd-fraction", "0.5", "--out", p("phys")])
    run(["gen", "--seed", "12", "--atoms", "2", "--lsph", "2", "--lnonsph", "1",
         "--basis-factor", "40", "--coeffs", "random", "--out", p("rand")])
    run(["build", p("phys"), "--out", p("phys_out")])
    run(["build", p("rand"), "--out", p("rand_out")])
