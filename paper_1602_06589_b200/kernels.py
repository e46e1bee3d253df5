"""The reference's level-3 operator plugin API, implemented on B200 tensor cores.

`KernelBackend` keeps the reference contract (`kernels.py:46-151`): argument
validation with `ContractViolationError`, nominal FLOP charging per call even for
empty shapes, Cholesky charged on success only, Hermitian/triangular operands read
from the lower triangle only, the strict upper triangle of a Hermitian target never
read.  `B200Kernels` executes every operator with the sm_100a kernels of
`libhsdla_b200.so` (DMMA contraction, batched Cholesky).  It is the single backend:
the reference's backend names ("optimized", "reference") are accepted as aliases so
`BuildConfig(backend=...)` values keep working, but there is no dispatch to any
other implementation and no CPU fallback.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native, device
from .errors import ConfigurationError, ContractViolationError, NotHPDError
from .matrix import ComplexDense, FlopLedger, HermitianAccumulator, cholesky_flops

_THREADS = 1


def set_thread_count(threads: int):
    """Validate and record the worker-thread cap (`kernels.py:33-38`).

    The reference caps BLAS threads; here the value is only echoed into the build
    report (`builder.py:421`), the GPU path needs no host threads."""
    global _THREADS
    if threads < 1:
        raise ConfigurationError(f"thread count must be >= 1, got {threads}")
    _THREADS = int(threads)


def _check(cond: bool, msg: str):
    if not cond:
        raise ContractViolationError(msg)


def _square_order(t: ComplexDense, role: str) -> int:
    _check(t.rows == t.cols, f"{role} is {t.rows}x{t.cols}; a square matrix is required")
    return t.rows


class KernelBackend:
    """The operator contract every backend shares (`kernels.py:46-132`): shapes are checked
    before anything runs, the nominal FLOPs of a call are charged whether or not the shape is
    empty, and a failed Cholesky charges nothing.  Subclasses supply the six `_xxx` workers."""

    name = "abstract"

    def __init__(self, threads: int = 1):
        self.threads = int(threads)
        set_thread_count(self.threads)

    # C (n x n, lower) += A^H A, A: k x n — 4 k n^2
    def hermitian_rank_k_update(self, c: HermitianAccumulator, a: ComplexDense,
                                ledger: FlopLedger) -> HermitianAccumulator:
        k, n = a.shape
        # both shapes in the message, target first (the reference's tests read them there)
        _check(c.n == n, f"ZHERK (rank-k) target {c.n}x{c.n} cannot take a {k}x{n} operand")
        if k > 0 and n > 0:
            self._herk(c.matrix, a)
        ledger.add("hermitian_rank_k", 4 * k * n * n)
        return c

    # C (n x n, lower) += X^H B + B^H X, X and B: k x n — 8 k n^2
    def hermitian_rank_2k_update(self, c: HermitianAccumulator, x: ComplexDense,
                                 b: ComplexDense, ledger: FlopLedger) -> HermitianAccumulator:
        _check(x.shape == b.shape, f"ZHER2K operands differ in shape: {x.shape} and {b.shape}")
        k, n = x.shape
        _check(c.n == n, f"ZHER2K (rank-2k) target {c.n}x{c.n} cannot take {k}x{n} operands")
        if k > 0 and n > 0:
            self._her2k(c.matrix, x, b)
        ledger.add("hermitian_rank_2k", 8 * k * n * n)
        return c

    # C = alpha op(A) B + beta C, op = conjugate transpose or identity — 8 m n k
    def general_product(self, c: ComplexDense, a: ComplexDense, b: ComplexDense,
                        conj_transpose_a: bool, alpha: complex, beta: complex,
                        ledger: FlopLedger) -> ComplexDense:
        m, k = (a.cols, a.rows) if conj_transpose_a else (a.rows, a.cols)
        n = b.cols
        _check(b.rows == k, f"ZGEMM contraction lengths disagree: op(A) gives {k}, B gives {b.rows}")
        _check(c.shape == (m, n), f"ZGEMM result is {m}x{n} but C is {c.rows}x{c.cols}")
        if m > 0 and n > 0:
            self._gemm(c, a, b, conj_transpose_a, complex(alpha), complex(beta))
        ledger.add("general_product", 8 * m * n * k)
        return c

    # X = alpha T A (+ X when accumulating), T Hermitian, lower triangle read — 8 n^2 cols
    def hermitian_product(self, x: ComplexDense, t: ComplexDense, a: ComplexDense,
                          accumulate: bool, alpha: complex,
                          ledger: FlopLedger) -> ComplexDense:
        n = _square_order(t, "the Hermitian operand")
        width = a.cols
        _check(a.rows == n, f"ZHEMM: T has order {n}, A has {a.rows} rows")
        _check(x.shape == (n, width), f"ZHEMM result is {n}x{width} but X is {x.rows}x{x.cols}")
        if n > 0 and width > 0:
            self._hemm(x, t, a, accumulate, complex(alpha))
        elif not accumulate:
            x.array[...] = 0.0
        ledger.add("hermitian_product", 8 * n * n * width)
        return x

    # Y = op(C) A, C lower triangular — 4 n^2 cols
    def triangular_product(self, y: ComplexDense, c: ComplexDense, a: ComplexDense,
                           conj_transpose_c: bool, ledger: FlopLedger) -> ComplexDense:
        n = _square_order(c, "the triangular factor")
        width = a.cols
        _check(a.rows == n, f"ZTRMM: factor has order {n}, A has {a.rows} rows")
        _check(y.shape == a.shape, f"ZTRMM result is {n}x{width} but Y is {y.rows}x{y.cols}")
        if n > 0 and width > 0:
            self._trmm(y, c, a, conj_transpose_c)
        ledger.add("triangular_product", 4 * n * n * width)
        return y

    def cholesky_factor(self, t: ComplexDense, ledger: FlopLedger) -> ComplexDense:
        """Lower Cholesky factor of T (its lower triangle is read) in a new matrix; T itself is
        never modified.  NotHPDError / ContractViolationError leave the ledger untouched."""
        n = _square_order(t, "the matrix to factor")
        factor = self._potrf(t)
        ledger.add("cholesky", cholesky_flops(n))
        return factor

    def _herk(self, c, a):  # pragma: no cover
        raise NotImplementedError

    def _her2k(self, c, x, b):  # pragma: no cover
        raise NotImplementedError

    def _gemm(self, c, a, b, conj_a, alpha, beta):  # pragma: no cover
        raise NotImplementedError

    def _hemm(self, x, t, a, accumulate, alpha):  # pragma: no cover
        raise NotImplementedError

    def _trmm(self, y, c, a, conj_c):  # pragma: no cover
        raise NotImplementedError

    def _potrf(self, t):  # pragma: no cover
        raise NotImplementedError


# -- the operators on numpy windows (column-major views with any leading dimension) -----------
# Shared by B200Kernels (this package's types) and the level-2 binding into the unmodified
# reference (integration.py), whose KernelBackend hands its private operators raw arrays.

def herk_lower(c: np.ndarray, a: np.ndarray):
    """lower(c) += a^H a (`kernels.py:242-244` zherk lower, trans=C), in place."""
    lib = _native.load()
    cd = device.upload_window(c)
    ad = device.upload_window(a)
    _native.check(lib.hsdla_herk_lower(device.ctx(), c.shape[0], a.shape[0], device.ptr(ad),
                                       ad.shape[1], device.ptr(cd), cd.shape[1]),
                  "hsdla_herk_lower")
    device.download_window(cd, c)


def her2k_lower(c: np.ndarray, x: np.ndarray, b: np.ndarray):
    """lower(c) += x^H b + b^H x (`kernels.py:246-248`), in place."""
    lib = _native.load()
    cd = device.upload_window(c)
    xd = device.upload_window(x)
    bd = device.upload_window(b)
    _native.check(lib.hsdla_her2k_lower(device.ctx(), c.shape[0], x.shape[0], device.ptr(xd),
                                        xd.shape[1], device.ptr(bd), bd.shape[1],
                                        device.ptr(cd), cd.shape[1]),
                  "hsdla_her2k_lower")
    device.download_window(cd, c)


def gemm(c: np.ndarray, a: np.ndarray, b: np.ndarray, conj_a: bool, alpha: complex, beta: complex):
    """c = alpha op(a) b + beta c (`kernels.py:250-253`), in place."""
    lib = _native.load()
    m, n = c.shape
    k = b.shape[0]
    ad = device.upload_window(a)
    bd = device.upload_window(b)
    cd = device.upload_window(c) if beta != 0 else device.empty_matrix(m, n)
    ws = device.empty_matrix(k, m) if not conj_a else None
    _native.check(lib.hsdla_gemm(device.ctx(), 1 if conj_a else 0, m, n, k,
                                 _native.c64(alpha), device.ptr(ad), ad.shape[1],
                                 device.ptr(bd), bd.shape[1], _native.c64(beta),
                                 device.ptr(cd), cd.shape[1],
                                 device.ptr(ws) if ws is not None else None),
                  "hsdla_gemm")
    device.download_window(cd, c)


def hemm_lower(x: np.ndarray, t: np.ndarray, a: np.ndarray, accumulate: bool, alpha: complex):
    """x = alpha herm(tril t) a (+ x) (`kernels.py:255-258`), in place."""
    lib = _native.load()
    m, n = x.shape
    td = device.upload_window(t)
    ad = device.upload_window(a)
    xd = device.upload_window(x) if accumulate else device.empty_matrix(m, n)
    ws = device.empty_matrix(m, m)
    _native.check(lib.hsdla_hemm_lower(device.ctx(), m, n, _native.c64(alpha), device.ptr(td),
                                       td.shape[1], device.ptr(ad), ad.shape[1],
                                       1 if accumulate else 0, device.ptr(xd), xd.shape[1],
                                       device.ptr(ws)),
                  "hsdla_hemm_lower")
    device.download_window(xd, x)


def trmm_lower(y: np.ndarray, c: np.ndarray, a: np.ndarray, conj_c: bool):
    """y = op(tril c) a (`kernels.py:260-264`), in place."""
    lib = _native.load()
    m, n = y.shape
    cdv = device.upload_window(c)
    ad = device.upload_window(a)
    yd = device.empty_matrix(m, n)
    ws = device.empty_matrix(m, m)
    _native.check(lib.hsdla_trmm_lower(device.ctx(), 1 if conj_c else 0, m, n, device.ptr(cdv),
                                       cdv.shape[1], device.ptr(ad), ad.shape[1],
                                       device.ptr(yd), yd.shape[1], device.ptr(ws)),
                  "hsdla_trmm_lower")
    device.download_window(yd, y)


def potrf_lower(t: np.ndarray) -> np.ndarray:
    """Lower Cholesky factor of tril(t) in a new array (`kernels.py:266-272`); t is not
    touched.  NotHPDError(pivot) / ContractViolationError (NaN) as the reference."""
    lib = _native.load()
    n = t.shape[0]
    if n == 0:
        return np.zeros((0, 0), dtype=np.complex128, order="F")
    td = device.upload_window(t)
    fd = device.empty_matrix(n, n)
    info = (ctypes.c_int32 * 1)()
    _native.check(lib.hsdla_potrf_lower_batched(device.ctx(), n, 1, device.ptr(td),
                                                td.shape[1], 0, device.ptr(fd), fd.shape[1],
                                                0, info),
                  "hsdla_potrf_lower_batched")
    if info[0] == -1:
        raise ContractViolationError("NaN in Cholesky input (lower triangle)")
    if info[0] > 0:
        raise NotHPDError(info[0] - 1)
    out = np.zeros((n, n), dtype=np.complex128, order="F")
    device.download_window(fd, out)
    return np.tril(out)


class B200Kernels(KernelBackend):
    """Every operator on the GPU: host windows are staged to HBM, computed by the
    sm_100a DMMA contraction / batched Cholesky, and copied back in place."""

    name = "b200"

    def _herk(self, c, a):
        herk_lower(c.array, a.array)

    def _her2k(self, c, x, b):
        her2k_lower(c.array, x.array, b.array)

    def _gemm(self, c, a, b, conj_a, alpha, beta):
        gemm(c.array, a.array, b.array, conj_a, alpha, beta)

    def _hemm(self, x, t, a, accumulate, alpha):
        hemm_lower(x.array, t.array, a.array, accumulate, alpha)

    def _trmm(self, y, c, a, conj_c):
        trmm_lower(y.array, c.array, a.array, conj_c)

    def _potrf(self, t):
        return ComplexDense(np.asfortranarray(potrf_lower(t.array)))


_ALIASES = {"b200": B200Kernels, "optimized": B200Kernels, "reference": B200Kernels}


def get_backend(name: str = "b200", threads: int = 1) -> KernelBackend:
    """Backend by name (`kernels.py:281-288`); reference names alias the B200 backend."""
    try:
        cls = _ALIASES[name]
    except KeyError:
        raise ConfigurationError(
            f"unknown backend {name!r}; choose from {sorted(_ALIASES)}") from None
    return cls(threads=threads)
