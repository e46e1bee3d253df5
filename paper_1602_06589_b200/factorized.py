"""Per-type phase-factorised H and S (FLEUR's FLOP reduction).

When the atoms of a type share rotation, radial data, muffin-tin radius, l_sph and T blocks,
every coefficient block is the type's template (the atom placed at the origin) times a
column phase (`flapw.py:220-231`):

    A_a[lm, G] = e^{i K_G . x_a} A^_t[lm, G],   likewise B_a, ||u_dot|| B_a, Z_a, Y_a, X_a,

so every stacked contraction of `build_all` (`builder.py:199-315`) splits per type into a
phase Gram and a template Gram multiplied elementwise:

    S = sum_t Phi_t o (A^_t^H A^_t + (U B^_t)^H (U B^_t))
    H = sum_t Phi_t o (Z^_t^H B^_t + B^_t^H Z^_t + Y^_t^H Y^_t   [or A^_t^H X^_t, non-HPD])
    Phi_t[G, G'] = sum_{a in t} conj(e_a(G)) e_a(G')

The work drops from O(N_A N_L N_G^2) to O(N_types (N_L + N_A/N_types) N_G^2): the template
Grams are the S and H of a one-atom system, built by the stacked pipeline itself; Phi_t is one
more DMMA contraction; the phases come from `hsdla_phase_matrix` and the combine is
`hsdla_hadamard_lower`.  Atoms are grouped into
types by exact equality of everything the coefficients depend on, so the result is always
the stacked build's (a system with no shared types gets one rank-1 phase Gram per atom).
This is an alternative evaluation, not `build_all`: the benchmark metric counts the
reference's stacked ledger.
"""
from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native, device
from .builder import BuildConfig, BuildReport, build_ledger, estimate_memory
from .errors import ContractViolationError
from .flapw import SystemSpec
from .matrix import AtomBlockLayout, ComplexDense


def atom_types(spec, tmats) -> list:
    """Groups of atom indices whose coefficient blocks differ only by the position phase:
    equal rotation, l_sph, muffin-tin radius, radial data and T blocks (by value)."""
    groups, keys = [], {}
    for a in range(spec.n_atoms):
        rad = spec.radial[a]
        key = (int(spec.l_sph[a]),
               np.asarray(spec.rotations[a], dtype=np.float64).tobytes(),
               float(spec.mt_radius[a]),
               b"".join(np.ascontiguousarray(getattr(rad, f), dtype=np.float64).tobytes()
                        for f in ("u", "u_prime", "udot", "udot_prime", "udot_norm")),
               b"".join(np.ascontiguousarray(t[a].array).tobytes()
                        for t in (tmats.t_aa, tmats.t_ab, tmats.t_bb)))
        if key not in keys:
            keys[key] = len(groups)
            groups.append([])
        groups[keys[key]].append(a)
    return groups


def _p(t, row0=0):
    return ctypes.c_void_p(t.data_ptr() + 16 * int(row0))


def build_hs_factorized(spec, tmats, config: BuildConfig | None = None):
    """(H, S, report) for one k-point through the per-type factorisation, H and S full
    Hermitian on the host (`ComplexDense`); report as `build_all`'s (reference ledger)."""
    t = device.require_cuda()
    t0 = time.perf_counter()
    h_d, s_d, mask, nbytes = build_hs_factorized_device(spec, tmats, config)
    n = int(spec.n_basis)
    hh = t.empty((max(n, 1), max(n, 1)), dtype=t.complex128, pin_memory=True)[:n, :n]
    hs = t.empty((max(n, 1), max(n, 1)), dtype=t.complex128, pin_memory=True)[:n, :n]
    hh.copy_(h_d[:n, :n])
    hs.copy_(s_d[:n, :n])
    wall = time.perf_counter() - t0
    config = config or BuildConfig()
    heights = [(int(l) + 1) ** 2 for l in spec.l_sph]
    layout = AtomBlockLayout(tuple(heights))
    sizes = [int(tmats.t_aa[a].rows) for a in range(spec.n_atoms)]
    report = BuildReport()
    report.ledger = build_ledger(heights, sizes, n, mask, config.force_general_path)
    report.hpd_mask = list(mask)
    report.hpd_atom_count = sum(mask)
    report.non_hpd_atom_count = len(mask) - sum(mask)
    report.timings = {"setup": wall, "S": 0.0, "H_ABBA_BB": 0.0, "H_AA": 0.0}
    report.predicted_bytes = estimate_memory(layout.atom_count, layout.capacity_block_height, n,
                                             config.backup)
    report.peak_observed_bytes = nbytes
    return ComplexDense(hh.numpy().T), ComplexDense(hs.numpy().T), report


def build_hs_factorized_device(spec, tmats, config: BuildConfig | None = None):
    """Device part of `build_hs_factorized`: (H, S) as (n, n) device tensors (row j = column
    j, full Hermitian), the HPD mask per atom and the device bytes used.

    Each type's template Grams come from the stacked pipeline run on a one-atom system (the
    type's atom at the origin): its S and H are exactly A^^H A^ + (U B^)^H (U B^) and
    Z^^H B^ + B^^H Z^ + Y^^H Y^ (or A^^H X^), with the T preparation, Cholesky dispatch and
    fused contractions of `hsdla_setup_hs`."""
    from .builder import TMatrixSet
    from .pipeline import DeviceSpec, HSPipeline, pack_tmats

    config = config or BuildConfig()
    t = device.require_cuda()
    lib = _native.load()
    c = device.ctx()
    n = int(spec.n_basis)
    groups = atom_types(spec, tmats)
    # phases, atoms in type order
    order = [a for g in groups for a in g]
    lde = max(16, -(-len(order) // 16) * 16)
    e_d = device.empty_matrix(lde, n, lde, zero=True)
    kv = t.from_numpy(np.ascontiguousarray(spec.k_vectors, dtype=np.float64)).cuda()
    pos = t.from_numpy(np.ascontiguousarray(np.asarray(spec.positions)[order], dtype=np.float64)).cuda()
    _native.check(lib.hsdla_phase_matrix(c, n, len(order), device.ptr(kv), device.ptr(pos),
                                         device.ptr(e_d), lde), "hsdla_phase_matrix")
    h_d = device.empty_matrix(n, n, n, zero=True)
    s_d = device.empty_matrix(n, n, n, zero=True)
    phi = device.empty_matrix(n, n, n)
    pipes = {}
    mask = [False] * spec.n_atoms
    e_row = 0
    for g in groups:
        rep = g[0]
        tspec = SystemSpec(positions=np.zeros((1, 3)),
                           rotations=np.asarray(spec.rotations)[[rep]],
                           mt_radius=np.asarray(spec.mt_radius)[[rep]],
                           l_sph=np.asarray(spec.l_sph)[[rep]],
                           l_nonsph=np.asarray(spec.l_nonsph)[[rep]], k_point=spec.k_point,
                           k_vectors=spec.k_vectors, omega=spec.omega, radial=[spec.radial[rep]])
        ttm = TMatrixSet([tmats.t_aa[rep]], [tmats.t_ab[rep]], [tmats.t_bb[rep]],
                         [tmats.l_sph[rep]], [tmats.l_nonsph[rep]])
        ds = DeviceSpec(tspec)
        key = int(ds.heights[0])
        if key not in pipes:
            pipes[key] = HSPipeline(n, ds.heights)
        pipe = pipes[key]
        res = pipe.run(ds, pack_tmats(ttm), config.force_general_path)
        for a in g:
            mask[a] = bool(res["hpd_mask"][0])
        # Phi_t = E_t^H E_t, then H += Phi_t o H_t, S += Phi_t o S_t (lower)
        phi.zero_()
        _native.check(lib.hsdla_herk_lower(c, n, len(g), _p(e_d, e_row), lde, device.ptr(phi), n),
                      "hsdla_herk_lower")
        e_row += len(g)
        for tmpl, acc in ((pipe.H, h_d), (pipe.S, s_d)):
            _native.check(lib.hsdla_hadamard_lower(c, n, device.ptr(phi), n, device.ptr(tmpl),
                                                   int(tmpl.shape[1]), device.ptr(acc), n, 1),
                          "hsdla_hadamard_lower")
    flag = ctypes.c_int32(0)
    for mat in (h_d, s_d):
        _native.check(lib.hsdla_mirror_lower(c, n, device.ptr(mat), n, ctypes.byref(flag)),
                      "hsdla_mirror_lower")
        if flag.value:
            raise ContractViolationError("accumulator contains non-finite values")
    nbytes = int(sum(x.numel() * x.element_size() for x in (e_d, h_d, s_d, phi)) +
                 sum(p.device_bytes for p in pipes.values()))
    return h_d, s_d, mask, nbytes
