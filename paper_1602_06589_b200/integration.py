"""Level-2 integration: the B200 operators as a `KernelBackend` inside the unmodified reference.

A maintainer who keeps the reference's own `builder.py` (`hsdla`, reference
`kernels.py:46-151`) and swaps only the level-3 operators registers this class into its
backend registry (`_BACKENDS`, `kernels.py:275-288`); `get_backend(name)` /
`BuildConfig(backend=name)` then run every ZHERK / ZHER2K / ZGEMM / ZHEMM / ZTRMM / ZPOTRF on
the sm_100a kernels.  The reference's `KernelBackend` keeps its validation and FLOP ledger and
hands the private operators raw numpy windows (`kernels.py:56-132`); the operators here are
`paper_1602_06589_b200.kernels.herk_lower` etc. on those arrays, with this package's
exceptions translated into the reference's own classes (its builder catches its NotHPDError,
`builder.py:285-288`).

    import hsdla                                   # the reference
    from paper_1602_06589_b200.integration import register_reference_backend
    register_reference_backend(hsdla)              # adds "b200"
    h, s, rep = hsdla.build_all(coeffs, tmats, hsdla.BuildConfig(backend="b200"))

Per-operator calls stage every operand across PCIe; the fused pipeline is
the fast path.  tests/test_ref_suite.py runs the reference's own test files through this.
"""
from __future__ import annotations

from . import kernels as _k
from .errors import ContractViolationError, NotHPDError


def reference_backend(hsdla):
    """The KernelBackend subclass of the given reference module bound to the B200 operators."""
    base = hsdla.kernels.KernelBackend
    ref_errors = hsdla.errors

    class B200ReferenceBackend(base):
        name = "b200"

        def _herk(self, c, a):
            _k.herk_lower(c, a)

        def _her2k(self, c, x, b):
            _k.her2k_lower(c, x, b)

        def _gemm(self, c, a, b, conj_a, alpha, beta):
            _k.gemm(c, a, b, conj_a, alpha, beta)

        def _hemm(self, x, t, a, accumulate, alpha):
            _k.hemm_lower(x, t, a, accumulate, alpha)

        def _trmm(self, y, c, a, conj_c):
            _k.trmm_lower(y, c, a, conj_c)

        def _potrf(self, lower):
            try:
                return _k.potrf_lower(lower)
            except NotHPDError as e:
                raise ref_errors.NotHPDError(e.pivot) from None
            except ContractViolationError as e:
                raise ref_errors.ContractViolationError(str(e)) from None

    return B200ReferenceBackend


def register_reference_backend(hsdla, names=("b200",)):
    """Register the B200 backend in the reference's registry under `names`; returns the class."""
    cls = reference_backend(hsdla)
    for n in names:
        hsdla.kernels._BACKENDS[n] = cls
    return cls
