"""Legendre-reduced A-side overlap on the GPU (drop-in for reference `oracle.py:159-216`
`ReducedOverlapInputs` / `reduced_S_AA` and `flapw.py:236-250` `reduced_overlap_inputs`).

By the addition theorem the m-sum of A*^H A* collapses to (2l+1)/(4 pi) P_l(cos), so the
A-side overlap needs O(N_A (l+1) N_G^2) work instead of the stacked contraction's
O(N_A (l+1)^2 N_G^2) (FLEUR's reduced overlap).  It is an
alternative evaluation of the A*^H A* part of S, not a replacement for the stacked build
(the benchmark metric counts the reference's stacked FLOP ledger).

* `reduced_overlap_inputs(spec)` computes the match factors with `hsdla_match_factors`
  (same Bessel code and rounding as the A/B generator);
* `reduced_S_AA(inputs)` runs `hsdla_reduced_s_aa` and returns the full Hermitian
  N_G x N_G matrix on the host; `reduced_S_AA_device` leaves it in HBM.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native, device
from .errors import ContractViolationError
from .matrix import ComplexDense


@dataclass
class ReducedOverlapInputs:
    """Factored inputs of the reduced A-side overlap (`oracle.py:159-183`): one real
    (l_a+1, N_G) match-factor array and one (l_a+1,) Wronskian array per atom."""

    f: list
    wronskians: list
    positions: np.ndarray
    k_vectors: np.ndarray
    omega: float

    def __post_init__(self):
        self.positions = np.asarray(self.positions, dtype=np.float64)
        self.k_vectors = np.asarray(self.k_vectors, dtype=np.float64)
        if self.omega <= 0:
            raise ContractViolationError("cell volume must be positive")
        if len(self.f) != len(self.wronskians) or len(self.f) != self.positions.shape[0]:
            raise ContractViolationError("per-atom input lists must align with positions")
        for w in self.wronskians:
            if np.any(np.asarray(w) == 0):
                raise ContractViolationError("zero Wronskian in reduced-overlap inputs")


def _rows(l_top):
    return np.concatenate(([0], np.cumsum(np.asarray(l_top, dtype=np.int64) + 1)[:-1])).astype(np.int64)


def reduced_overlap_inputs(spec) -> ReducedOverlapInputs:
    """Match factors f_A per atom computed on the GPU (`flapw.py:236-250`)."""
    from .pipeline import DeviceSpec

    t = device.require_cuda()
    lib = _native.load()
    ds = DeviceSpec(spec)
    l_top = ds.l_sph.astype(np.int32)
    f_row = _rows(l_top)
    n = ds.n_basis
    fa = t.empty((int((l_top + 1).sum()), n), dtype=t.float64, device="cuda")
    args = _native.AbArgs()
    args.n_atoms, args.n_basis = ds.n_atoms, n
    args.k_vectors, args.positions = ds.kv.data_ptr(), ds.pos.data_ptr()
    args.rotations, args.mt_radius = ds.rot.data_ptr(), ds.rmt.data_ptr()
    args.radial, args.radial_stride = ds.radial.data_ptr(), ds.radial_stride
    args.l_sph = l_top.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    args.omega = ds.omega
    _native.check(lib.hsdla_match_factors(device.ctx(), ctypes.byref(args),
                                          f_row.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                          device.ptr(fa), None, n), "hsdla_match_factors")
    host = fa.cpu().numpy()
    f = [host[r:r + int(l) + 1].copy() for r, l in zip(f_row, l_top)]
    w = [np.asarray(spec.radial[a].wronskian)[: int(l_top[a]) + 1] for a in range(ds.n_atoms)]
    return ReducedOverlapInputs(f=f, wronskians=w, positions=spec.positions,
                                k_vectors=spec.k_vectors, omega=spec.omega)


class ReducedPlan:
    """Inputs of `hsdla_reduced_s_aa` staged in HBM once; `run` is the kernel launch alone.

    Atoms with identical match factors and Wronskians (one atom type) share f rows; the
    kernel then evaluates their radial sum once and only the phases per atom."""

    def __init__(self, inputs: ReducedOverlapInputs):
        t = device.require_cuda()
        self.n = n = int(inputs.k_vectors.shape[0])
        self.l_top = np.array([fa.shape[0] - 1 for fa in inputs.f], dtype=np.int32)
        if self.l_top.max(initial=0) > _native.MAX_LSPH:
            raise ContractViolationError(f"l > {_native.MAX_LSPH} is not compiled in")
        uniq, self.f_row = {}, np.zeros(len(inputs.f), dtype=np.int64)
        blocks, coef, nrow = [], [], 0
        for a, (fa, w) in enumerate(zip(inputs.f, inputs.wronskians)):
            fa = np.ascontiguousarray(fa, dtype=np.float64)
            if fa.shape[1] != n:
                raise ContractViolationError("match factors must have one column per K-vector")
            w = np.asarray(w, dtype=np.float64)
            key = (fa.shape, fa.tobytes(), w[: fa.shape[0]].tobytes())
            if key not in uniq:
                uniq[key] = nrow
                blocks.append(fa)
                # (2l+1) / (4 pi) / W_l^2 per row, the reference's scalar expression (oracle.py:209)
                coef += [(2 * l + 1) / (4.0 * np.pi) / (w[l] ** 2) for l in range(fa.shape[0])]
                nrow += fa.shape[0]
            self.f_row[a] = uniq[key]
        self.n_types = len(blocks)
        host = (np.ascontiguousarray(inputs.k_vectors), np.ascontiguousarray(inputs.positions),
                np.ascontiguousarray(np.concatenate(blocks)), np.asarray(coef, dtype=np.float64))
        self.kv, self.pos, self.f, self.coef = (t.from_numpy(x).to("cuda") for x in host)
        self.n_atoms = len(inputs.f)
        self.scale = (4.0 * np.pi) ** 2 / inputs.omega

    def run(self, out=None):
        t = device.torch()
        lib = _native.load()
        n = self.n
        if out is None:
            out = t.empty((max(n, 1), max(n, 1)), dtype=t.complex128, device="cuda")
        a = _native.ReducedArgs()
        a.n_atoms, a.n_basis = self.n_atoms, n
        a.k_vectors, a.positions = self.kv.data_ptr(), self.pos.data_ptr()
        a.f, a.coef, a.ld_f = self.f.data_ptr(), self.coef.data_ptr(), n
        a.f_row = self.f_row.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        a.l_top = self.l_top.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        a.scale = self.scale
        a.S = out.data_ptr()
        a.lds = int(out.shape[1])
        _native.check(lib.hsdla_reduced_s_aa(device.ctx(), ctypes.byref(a)), "hsdla_reduced_s_aa")
        return out


def reduced_S_AA_device(inputs: ReducedOverlapInputs, out=None):
    """Reduced A-side overlap into HBM: a (N_G, N_G) complex128 tensor, row j = column j."""
    return ReducedPlan(inputs).run(out)


def reduced_S_AA(inputs: ReducedOverlapInputs) -> ComplexDense:
    """A-side overlap through the Legendre-reduced m-free sum (`oracle.py:186-216`)."""
    n = int(inputs.k_vectors.shape[0])
    dev = reduced_S_AA_device(inputs)
    host = dev[:n, :n].cpu().numpy()   # (column, row) storage
    return ComplexDense(np.asfortranarray(host.T))
