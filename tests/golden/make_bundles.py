"""Golden bundles: run the REAL reference CLI (build container only).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_bundles.py

Writes under tests/golden/bundles/:
* phys/      `hsdla gen --seed 11 --atoms 4 --lsph 3 --lnonsph 2 --basis-factor 50
               --hpd-fraction 0.5` (physics coefficients, system.json, 2 HPD + 2 non-HPD atoms)
* phys_out/  `hsdla build phys` (H.hsm1, S.hsm1, report.json)
* rand/      `hsdla gen --seed 12 --atoms 2 --lsph 2 --lnonsph 1 --basis-factor 40
               --coeffs random` (no system.json)
* rand_out/  `hsdla build rand`
* small/      `hsdla gen --seed 13 --atoms 2 --lsph 2 --lnonsph 1 --basis-factor 6
               --coeffs random` (2R >= N_G: verify runs the S Cholesky check)
* phys_verify/, rand_verify/, small_verify/  `hsdla verify` of each (verify.json; exit 0)
* phys_fault/ phys with T_BB of atom 0 de-Hermitised (SPEC.md:491's injected fault; the
               manifest hash updated), phys_fault_verify/ its `hsdla verify` (exit 4, the
               oracle's Hermitian residual of H flagged) and exit_code.txt
These pin `paper_1602_06589_b200.bundle.build_bundle`, the `verify` command and the HSM1
reader/writer (tests/test_bundle.py, tests/test_gpu_verify.py).
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
    run(["gen", "--seed", "13", "--atoms", "2", "--lsph", "2", "--lnonsph", "1",
         "--basis-factor", "6", "--coeffs", "random", "--out", p("small")])
    run(["verify", p("small"), "--out", p("small_verify")])
    run(["verify", p("phys"), "--out", p("phys_verify")])
    run(["verify", p("rand"), "--out", p("rand_verify")])
    # injected fault: T_BB of atom 0 de-Hermitised (upper triangle perturbed, lower kept)
    import hashlib
    import json

    import numpy as np
    from hsdla.matrix import ComplexDense, read_hsm1, write_hsm1

    shutil.copytree(p("phys"), p("phys_fault"))
    tbb = read_hsm1(os.path.join(p("phys_fault"), "T_BB_000.hsm1")).array.copy()
    iu = np.triu_indices(tbb.shape[0], 1)
    tbb[iu] += 0.25 + 0.5j
    write_hsm1(os.path.join(p("phys_fault"), "T_BB_000.hsm1"), ComplexDense.from_array(tbb))
    man = json.loads(open(os.path.join(p("phys_fault"), "manifest.json")).read())
    with open(os.path.join(p("phys_fault"), "T_BB_000.hsm1"), "rb") as fh:
        man["files"]["T_BB_000.hsm1"] = "sha256:" + hashlib.sha256(fh.read()).hexdigest()
    open(os.path.join(p("phys_fault"), "manifest.json"), "w").write(json.dumps(man, sort_keys=True, indent=1))
    rc = main(["verify", p("phys_fault"), "--out", p("phys_fault_verify")])
    open(os.path.join(p("phys_fault_verify"), "exit_code.txt"), "w").write(f"{rc}\n")
    assert rc == 4, rc
