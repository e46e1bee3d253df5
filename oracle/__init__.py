"""CPU oracle for the muffin-tin H/S setup path — TEST INFRASTRUCTURE ONLY.

This package is a plain numpy/scipy restatement of the reference `hsdla`
algorithm (arXiv 1602.06589 HSDLA; reference package under
`pkg/src/hsdla/`), written from the reference's behaviour, not copied from it.
Every function cites the reference file:line it restates.

Who may use it: `tests/`, `__graft_entry__.smoke()` (as the checker) and
`bench.py` (the `cpu_baseline` leg and `--impl reference`).  The product
package `paper_1602_06589_b200` never imports it: the product path runs on
the GPU through `libhsdla_b200.so` and fails loudly when that is missing.

Parity pinning: `tests/golden/make_golden.py` runs the real reference (from
/root/reference, in the build container) on seeded inputs and stores golden
vectors under `tests/golden/`; `tests/test_oracle_golden.py` checks this
oracle against them.
"""
