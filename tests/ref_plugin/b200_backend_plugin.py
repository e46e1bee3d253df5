"""pytest plugin (test infrastructure): run the UNMODIFIED reference package's own tests with the
B200 operators registered as its KernelBackend (level 2).

Loaded with `-p b200_backend_plugin` and the reference (baseline/_ref) first on sys.path: every
backend name the reference's tests ask for ("reference", "optimized") resolves to
`paper_1602_06589_b200.integration.reference_backend(hsdla)`, the reference-side binding a
maintainer would add, so the reference's own builder drives the sm_100a operators."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if REPO not in sys.path:
    sys.path.append(REPO)


def pytest_configure(config):
    import hsdla

    from paper_1602_06589_b200.integration import register_reference_backend

    register_reference_backend(hsdla, names=("b200", "reference", "optimized"))
