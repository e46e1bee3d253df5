"""HSM1 matrix files (drop-in for reference `matrix.py:242-276`) and their HBM streaming path.

Format (`matrix.py:18`, `:242-250`): the 8-byte magic ``b"HSDLAM1\\x00"``, rows and cols
as little-endian uint64, then rows*cols little-endian complex128 values in column-major
order, always compacted (ld == rows).

* `write_hsm1` / `read_hsm1` keep the reference signatures, messages and exceptions for
  host `ComplexDense` windows.
* `write_hsm1_device` / `read_hsm1_device` are the B200 path for H, S, A*, B*: the matrix
  stays in HBM and moves through two pinned panels, so the PCIe copy of panel i+1
  overlaps the file write (or read) of panel i and no full host copy is ever made.  The
  non-finite guard runs in HBM (`hsdla_check_finite`).
"""
from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

from . import _native, device
from .errors import ContractViolationError
from .matrix import ComplexDense

HSM1_MAGIC = b"HSDLAM1\x00"
_HEADER = struct.Struct("<QQ")
_PANEL_BYTES = 32 << 20


def write_hsm1(path, m: ComplexDense) -> None:
    """Write a matrix in the HSM1 binary format (compacted to ld == rows), `matrix.py:242-250`."""
    a = m.array
    if not np.isfinite(a).all():
        raise ContractViolationError("refusing to serialize non-finite values")
    with open(path, "wb") as fh:
        fh.write(HSM1_MAGIC)
        fh.write(_HEADER.pack(m.rows, m.cols))
        fh.write(np.asfortranarray(a).astype("<c16", copy=False).tobytes(order="F"))


def _read_header(fh, path):
    magic = fh.read(8)
    if magic != HSM1_MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}, not an HSM1 file")
    header = fh.read(_HEADER.size)
    if len(header) != _HEADER.size:
        raise ValueError(f"{path}: truncated HSM1 header")
    return _HEADER.unpack(header)


def _payload_check(path, got: int, rows: int, cols: int) -> None:
    expected = 16 * rows * cols
    if got != expected:
        raise ValueError(f"{path}: payload is {got} bytes, expected {expected} "
                         f"for a {rows}x{cols} matrix")


def read_hsm1(path) -> ComplexDense:
    """Read a matrix from the HSM1 binary format, `matrix.py:253-276`."""
    with open(path, "rb") as fh:
        rows, cols = _read_header(fh, path)
        payload = fh.read()
    _payload_check(path, len(payload), rows, cols)
    if rows == 0 or cols == 0:
        return ComplexDense(np.zeros((rows, cols), dtype=np.complex128, order="F"))
    flat = np.frombuffer(payload, dtype="<c16")
    return ComplexDense(np.asfortranarray(flat.reshape((rows, cols), order="F")
                                          .astype(np.complex128)))


def _panel_cols(rows: int, cols: int, panel_bytes: int) -> int:
    return max(1, min(cols, panel_bytes // max(16 * rows, 1)))


def write_hsm1_device(path, dev, rows: int, cols: int | None = None, *,
                      panel_bytes: int = _PANEL_BYTES) -> int:
    """Stream an HBM-resident column-major window to an HSM1 file; returns bytes written.

    `dev` is a device tensor of shape (cols, ld) (row j = column j, as everywhere in this
    package) holding the matrix in its first `rows` entries per column.  Raises
    ContractViolationError, before creating the file, if any element is NaN or Inf."""
    t = device.require_cuda()
    lib = _native.load()
    cols = int(dev.shape[0]) if cols is None else int(cols)
    ld = int(dev.shape[1])
    rows = int(rows)
    if rows > ld or cols > dev.shape[0]:
        raise ContractViolationError(f"window {rows}x{cols} exceeds the device buffer")
    bad = ctypes.c_int32(0)
    _native.check(lib.hsdla_check_finite(device.ctx(), rows, cols, device.ptr(dev), max(ld, 1),
                                         ctypes.byref(bad)), "hsdla_check_finite")
    if bad.value:
        raise ContractViolationError("refusing to serialize non-finite values")
    with open(path, "wb") as fh:
        fh.write(HSM1_MAGIC)
        fh.write(_HEADER.pack(rows, cols))
        if rows == 0 or cols == 0:
            return fh.tell()
        pc = _panel_cols(rows, cols, panel_bytes)
        bufs = [t.empty((pc, rows), dtype=t.complex128, pin_memory=True) for _ in range(2)]
        done = [t.cuda.Event(), t.cuda.Event()]
        copy = t.cuda.Stream()
        copy.wait_stream(t.cuda.current_stream())
        dev.record_stream(copy)
        starts = list(range(0, cols, pc))

        def enqueue(i):
            c0 = starts[i]
            c1 = min(cols, c0 + pc)
            with t.cuda.stream(copy):
                bufs[i % 2][:c1 - c0].copy_(dev[c0:c1, :rows], non_blocking=True)
                done[i % 2].record(copy)

        enqueue(0)
        for i, c0 in enumerate(starts):
            if i + 1 < len(starts):
                enqueue(i + 1)  # its buffer was written out in iteration i - 1
            done[i % 2].synchronize()
            c1 = min(cols, c0 + pc)
            fh.write(memoryview(bufs[i % 2][:c1 - c0].numpy()).cast("B"))
        return fh.tell()


def read_hsm1_device(path, ld: int | None = None, *, panel_bytes: int = _PANEL_BYTES):
    """Read an HSM1 file straight into HBM: returns (device tensor (cols, ld), rows, cols).

    Rows rows..ld-1 of the returned buffer are zero.  Header and size errors are the
    reference's ValueErrors (`matrix.py:253-270`)."""
    t = device.require_cuda()
    with open(path, "rb") as fh:
        rows, cols = _read_header(fh, path)
        _payload_check(path, os.fstat(fh.fileno()).st_size - 8 - _HEADER.size, rows, cols)
        ld = max(rows, 1) if ld is None else int(ld)
        if ld < rows:
            raise ContractViolationError(f"ld {ld} < rows {rows}")
        dev = device.empty_matrix(rows, cols, ld, zero=ld > rows or rows == 0)
        if rows == 0 or cols == 0:
            return dev, rows, cols
        pc = _panel_cols(rows, cols, panel_bytes)
        bufs = [t.empty((pc, rows), dtype=t.complex128, pin_memory=True) for _ in range(2)]
        done = [None, None]
        copy = t.cuda.Stream()
        copy.wait_stream(t.cuda.current_stream())
        for i, c0 in enumerate(range(0, cols, pc)):
            c1 = min(cols, c0 + pc)
            k = i % 2
            if done[k] is not None:
                done[k].synchronize()  # the H2D that last used this buffer has finished
            view = memoryview(bufs[k][:c1 - c0].numpy()).cast("B")
            if fh.readinto(view) != len(view):
                raise ValueError(f"{path}: payload ended early")
            with t.cuda.stream(copy):
                dev[c0:c1, :rows].copy_(bufs[k][:c1 - c0], non_blocking=True)
                done[k] = t.cuda.Event()
                done[k].record(copy)
        t.cuda.current_stream().wait_stream(copy)
        for e in done:
            if e is not None:
                e.synchronize()  # pinned panels are released on return
        return dev, rows, cols
