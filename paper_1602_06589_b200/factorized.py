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

The work drops from O(N_A N_L N_G^2) to O(N_types (N_L + N_A/N_types) N_G^2): every Gram is
the same sm_100a DMMA contraction (`hsdla_herk_lower` / `her2k` / `gemm`), the phases come
from `hsdla_phase_matrix` and the combine is `hsdla_hadamard_lower`.  Atoms are grouped into
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
    j, full Hermitian), the HPD mask per atom and the device bytes used."""
    from .pipeline import DeviceSpec, ab_generate_device, padded_ld

    config = config or BuildConfig()
    t = device.require_cuda()
    lib = _native.load()
    c = device.ctx()
    n = int(spec.n_basis)
    groups = atom_types(spec, tmats)
    reps = [g[0] for g in groups]
    # templates: one atom per type at the origin (same rotation / radial data / radius)
    tspec = SystemSpec(positions=np.zeros((len(reps), 3)),
                       rotations=np.asarray(spec.rotations)[reps],
                       mt_radius=np.asarray(spec.mt_radius)[reps],
                       l_sph=np.asarray(spec.l_sph)[reps], l_nonsph=np.asarray(spec.l_nonsph)[reps],
                       k_point=spec.k_point, k_vectors=spec.k_vectors, omega=spec.omega,
                       radial=[spec.radial[a] for a in reps])
    ds = DeviceSpec(tspec)
    ld = padded_ld(ds.rows)
    a_d = device.empty_matrix(ld, n, ld, zero=True)
    b_d = device.empty_matrix(ld, n, ld, zero=True)
    bs_d = device.empty_matrix(ld, n, ld, zero=True)
    ab_generate_device(ds, a_d, b_d, bs_d, ld, None)
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
    gram = device.empty_matrix(n, n, n)
    mask = [False] * spec.n_atoms
    e_row = 0
    for ti, g in enumerate(groups):
        rep = g[0]
        h = int(ds.heights[ti])
        r0 = int(ds.row_offset[ti])
        m = int(tmats.t_aa[rep].rows)
        # Phi_t = E_t^H E_t
        phi.zero_()
        _native.check(lib.hsdla_herk_lower(c, n, len(g), _p(e_d, e_row), lde, device.ptr(phi), n),
                      "hsdla_herk_lower")
        e_row += len(g)
        # S: A^^H A^ + (U B^)^H (U B^)
        gram.zero_()
        _native.check(lib.hsdla_herk_lower(c, n, h, _p(a_d, r0), ld, device.ptr(gram), n), "herk")
        _native.check(lib.hsdla_herk_lower(c, n, h, _p(bs_d, r0), ld, device.ptr(gram), n), "herk")
        _native.check(lib.hsdla_hadamard_lower(c, n, device.ptr(phi), n, device.ptr(gram), n,
                                               device.ptr(s_d), n, 1), "hsdla_hadamard_lower")
        if m == 0:
            continue
        # H: Z^ = T_AB^H A^ + 1/2 T_BB B^ on the first m rows, then Z^^H B^ + B^^H Z^
        tab = device.upload_window(tmats.t_ab[rep].array)
        tbb = device.upload_window(tmats.t_bb[rep].array)
        taa = device.upload_window(tmats.t_aa[rep].array)
        ws = device.empty_matrix(m, m)
        z_d = device.empty_matrix(m, n, m)
        _native.check(lib.hsdla_gemm(c, 1, m, n, m, _native.c64(1.0), device.ptr(tab), tab.shape[1],
                                     _p(a_d, r0), ld, _native.c64(0.0), device.ptr(z_d), m, None),
                      "hsdla_gemm")
        _native.check(lib.hsdla_hemm_lower(c, m, n, _native.c64(0.5), device.ptr(tbb), tbb.shape[1],
                                           _p(b_d, r0), ld, 1, device.ptr(z_d), m, device.ptr(ws)),
                      "hsdla_hemm_lower")
        gram.zero_()
        _native.check(lib.hsdla_her2k_lower(c, n, m, device.ptr(z_d), m, _p(b_d, r0), ld,
                                            device.ptr(gram), n), "hsdla_her2k_lower")
        # AA: Cholesky per type (builder.py:274-315): Y^ = C^H A^ (HPD) or X^ = T_AA A^
        fac = device.empty_matrix(m, m)
        info = (ctypes.c_int32 * 1)()
        hpd = False
        if not config.force_general_path:
            _native.check(lib.hsdla_potrf_lower_batched(c, m, 1, device.ptr(taa), taa.shape[1], 0,
                                                        device.ptr(fac), m, 0, info), "potrf")
            if info[0] == -1:
                raise ContractViolationError("NaN in Cholesky input (lower triangle)")
            hpd = info[0] == 0
        xy = device.empty_matrix(m, n, m)
        if hpd:
            _native.check(lib.hsdla_trmm_lower(c, 1, m, n, device.ptr(fac), m, _p(a_d, r0), ld,
                                               device.ptr(xy), m, device.ptr(ws)), "hsdla_trmm_lower")
            _native.check(lib.hsdla_herk_lower(c, n, m, device.ptr(xy), m, device.ptr(gram), n),
                          "hsdla_herk_lower")
        else:
            _native.check(lib.hsdla_hemm_lower(c, m, n, _native.c64(1.0), device.ptr(taa),
                                               taa.shape[1], _p(a_d, r0), ld, 0, device.ptr(xy), m,
                                               device.ptr(ws)), "hsdla_hemm_lower")
            _native.check(lib.hsdla_gemm(c, 1, n, n, m, _native.c64(1.0), _p(a_d, r0), ld,
                                         device.ptr(xy), m, _native.c64(1.0), device.ptr(gram), n,
                                         None), "hsdla_gemm")
        for a in g:
            mask[a] = hpd
        _native.check(lib.hsdla_hadamard_lower(c, n, device.ptr(phi), n, device.ptr(gram), n,
                                               device.ptr(h_d), n, 1), "hsdla_hadamard_lower")
    flag = ctypes.c_int32(0)
    for mat in (h_d, s_d):
        _native.check(lib.hsdla_mirror_lower(c, n, device.ptr(mat), n, ctypes.byref(flag)),
                      "hsdla_mirror_lower")
        if flag.value:
            raise ContractViolationError("accumulator contains non-finite values")
    nbytes = int(sum(x.numel() * x.element_size()
                     for x in (a_d, b_d, bs_d, e_d, h_d, s_d, phi, gram)))
    return h_d, s_d, mask, nbytes
