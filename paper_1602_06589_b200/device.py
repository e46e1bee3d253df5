"""Device plumbing: CUDA context per stream, HBM buffers, host<->device staging.

PyTorch is used for device memory, streams and pinned host memory only; every
computation goes through `libhsdla_b200.so`.  Column-major complex128 matrices
live in torch tensors of shape (cols, ld): row j of the tensor is column j of the
matrix, so `data_ptr()` is exactly the column-major base pointer the C ABI takes.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import ContractViolationError, NativeLibraryError

_torch = None
_CTX = {}


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise NativeLibraryError(
            "no CUDA device visible: the H/S path runs only on the GPU (no CPU fallback)")
    return t


def ctx():
    """The libhsdla context bound to torch's current CUDA stream on the current device."""
    t = require_cuda()
    lib = _native.load()
    dev = t.cuda.current_device()
    stream = t.cuda.current_stream(dev).cuda_stream
    c = _CTX.get(dev)
    if c is None:
        handle = ctypes.c_void_p()
        _native.check(lib.hsdla_ctx_create(ctypes.byref(handle), ctypes.c_void_p(stream)),
                      "hsdla_ctx_create")
        c = [handle, stream]
        _CTX[dev] = c
    elif c[1] != stream:
        _native.check(lib.hsdla_ctx_set_stream(c[0], ctypes.c_void_p(stream)), "hsdla_ctx_set_stream")
        c[1] = stream
    return c[0]


def empty_matrix(rows: int, cols: int, ld: int | None = None, zero: bool = False):
    """Device column-major complex128 matrix (tensor of shape (cols, ld))."""
    t = require_cuda()
    ld = max(rows, 1) if ld is None else ld
    shape = (max(cols, 1), ld)
    if zero:
        return t.zeros(shape, dtype=t.complex128, device="cuda")
    return t.empty(shape, dtype=t.complex128, device="cuda")


def ptr(tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(tensor.data_ptr())


def upload_window(host: np.ndarray, ld: int | None = None, pinned: bool = False):
    """Copy a (rows, cols) numpy window (any strides) to a device (cols, ld) tensor."""
    t = require_cuda()
    rows, cols = host.shape
    ld = max(rows, 1) if ld is None else ld
    dev = empty_matrix(rows, cols, ld)
    if rows and cols:
        src = t.from_numpy(np.ascontiguousarray(host.T))
        if pinned:
            src = src.pin_memory()
        dev[:cols, :rows].copy_(src, non_blocking=pinned)
    return dev


def pinned_stack(rows: int, cols: int, capacity_rows: int):
    """Host column-major (capacity_rows x cols) complex128 allocation in pinned memory (torch's
    caching host allocator), as the F-ordered numpy base of a `ComplexDense` window of `rows`
    rows, plus its (cols, capacity_rows) tensor view for whole-buffer copies."""
    t = torch()
    buf = t.empty((max(cols, 1), max(capacity_rows, 1)), dtype=t.complex128, pin_memory=True)
    return buf.numpy().T[:capacity_rows, :cols], buf


def upload_stack(window, ld_min: int | None = None):
    """Device (cols, ld) copy of a stacked-coefficient window.  A window at the top of an
    F-ordered allocation (the layout `compute_AB` returns) goes up as one contiguous copy of
    the whole allocation (ld = its capacity height; pinned memory makes it a DMA at full
    PCIe speed) when that height keeps 16-element (256-byte) K-chunk alignment and is at least
    `ld_min`; anything else is packed first (ld = `ld_min` or the window height)."""
    t = require_cuda()
    base = window.base
    rows, cols = window.shape
    if (window.row_offset == 0 and base.flags.f_contiguous and base.shape[1] == cols
            and base.shape[0] >= max(rows, 1)
            and (ld_min is None or (base.shape[0] >= ld_min and base.shape[0] % 16 == 0))):
        dev = t.from_numpy(base.T).to("cuda", non_blocking=True)
        return dev, int(base.shape[0])
    ld = ld_min or max(rows, 1)
    return upload_window(window.array, ld), ld


def pinned_sources(a_window, b_window):
    """(A_host, B_host, ld) when both stacked windows start at row 0 of F-ordered complex128
    allocations of the same height that live in pinned host memory (the layout `compute_AB`
    returns), so the native build can DMA them itself; else None."""
    lib = _native.load()
    ptrs = []
    ld = None
    for w in (a_window, b_window):
        base = w.base
        if (w.row_offset != 0 or base.dtype != np.complex128 or not base.flags.f_contiguous
                or base.shape[1] != w.cols or (ld is not None and base.shape[0] != ld)):
            return None
        ld = int(base.shape[0])
        p = base.ctypes.data
        if not lib.hsdla_is_pinned(ctypes.c_void_p(p)):
            return None
        ptrs.append(p)
    return ptrs[0], ptrs[1], ld


def download_window(dev, out: np.ndarray):
    """Copy the device (cols, ld) tensor's leading rows into the numpy window `out`."""
    rows, cols = out.shape
    if rows and cols:
        if out.flags.f_contiguous and out.dtype == np.complex128:
            torch().from_numpy(out.T).copy_(dev[:cols, :rows])  # one copy, straight into `out`
        else:
            out[...] = dev[:cols, :rows].cpu().numpy().T


def upload_real(vec) -> object:
    t = require_cuda()
    return t.from_numpy(np.ascontiguousarray(np.asarray(vec, dtype=np.float64))).to("cuda")


def mirror_host_inplace(m) -> None:
    """HermitianAccumulator.mirror_to_full on the GPU (matrix.py:216-226)."""
    n = m.rows
    if n == 0:
        return
    dev = upload_window(m.array)
    flag = ctypes.c_int32(0)
    lib = _native.load()
    _native.check(lib.hsdla_mirror_lower(ctx(), n, ptr(dev), dev.shape[1], ctypes.byref(flag)),
                  "hsdla_mirror_lower")
    download_window(dev, m.array)
    if flag.value:
        raise ContractViolationError("accumulator contains non-finite values")


def scale_rows_host_inplace(b, d: np.ndarray) -> None:
    """scale_rows on the GPU (matrix.py:229-239)."""
    if b.rows == 0 or b.cols == 0:
        return
    dev = upload_window(b.array)
    dd = upload_real(d)
    lib = _native.load()
    _native.check(lib.hsdla_scale_rows(ctx(), b.rows, b.cols, ptr(dd), ptr(dev), dev.shape[1]),
                  "hsdla_scale_rows")
    download_window(dev, b.array)
