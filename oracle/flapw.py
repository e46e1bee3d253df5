"""Oracle restatement of the matching-coefficient generation (test infrastructure).

`compute_ab(spec)` follows reference `flapw.py:201-233` (compute_AB) with
`match_factors` (`flapw.py:179-198`) and `_unit_directions` (`flapw.py:169-176`),
vectorised over the K-vectors.  `spec` is duck-typed: any object with the
`SystemSpec` fields (`flapw.py:85-166`) works, including the reference's own.
Returns plain numpy arrays: A, B of shape (R, N_G) complex128 (rows per atom in
(l, m) order l^2 + l + m), the per-row ||u_dot|| (R,) and the row offsets.
"""
from __future__ import annotations

import numpy as np

from .special import spherical_bessel_all, spherical_harmonics_all


def unit_directions(k_vectors: np.ndarray):
    """|K| and K/|K|, the zero vector mapped to +z (`flapw.py:169-176`)."""
    norms = np.linalg.norm(k_vectors, axis=1)
    unit = np.zeros_like(k_vectors)
    nz = norms > 0
    unit[nz] = k_vectors[nz] / norms[nz, None]
    unit[~nz] = (0.0, 0.0, 1.0)
    return norms, unit


def wronskian(rad) -> np.ndarray:
    """W_l = udot * u' - u * udot' (`flapw.py:62-64`)."""
    return np.asarray(rad.udot) * np.asarray(rad.u_prime) - np.asarray(rad.u) * np.asarray(rad.udot_prime)


def match_factors(spec, atom: int, columns=None):
    """(f_A, f_B), each (l_sph+1, n) real (`flapw.py:179-198`)."""
    rad = spec.radial[atom]
    l_top = int(spec.l_sph[atom])
    r_mt = float(spec.mt_radius[atom])
    kv = np.asarray(spec.k_vectors, dtype=np.float64)
    if columns is not None:
        kv = kv[columns]
    norms, _ = unit_directions(kv)
    j, jp = spherical_bessel_all(l_top, r_mt * norms)
    sl = slice(0, l_top + 1)
    udot, udot_p = np.asarray(rad.udot)[sl], np.asarray(rad.udot_prime)[sl]
    u, u_p = np.asarray(rad.u)[sl], np.asarray(rad.u_prime)[sl]
    f_a = udot[:, None] * norms[None, :] * jp - udot_p[:, None] * j
    f_b = -u[:, None] * norms[None, :] * jp + u_p[:, None] * j
    return f_a, f_b


def row_offsets(spec) -> np.ndarray:
    heights = [(int(l) + 1) ** 2 for l in spec.l_sph]
    return np.concatenate(([0], np.cumsum(heights))).astype(np.int64)


def compute_ab(spec, columns=None):
    """A, B, udot_norms, offsets for the stacked atoms (`flapw.py:201-233`).

    `columns` optionally restricts the evaluation to a subset of K-vectors
    (used by full-size parity tests that check sampled columns).
    """
    kv = np.asarray(spec.k_vectors, dtype=np.float64)
    if columns is not None:
        kv = kv[columns]
    n = kv.shape[0]
    offs = row_offsets(spec)
    r = int(offs[-1])
    a_star = np.zeros((r, n), dtype=np.complex128)
    b_star = np.zeros((r, n), dtype=np.complex128)
    udot_norms = np.zeros(r)
    _, unit = unit_directions(kv)
    omega = float(spec.omega)
    for a in range(len(spec.l_sph)):
        rad = spec.radial[a]
        l_top = int(spec.l_sph[a])
        w = wronskian(rad)
        rot = np.asarray(spec.rotations[a], dtype=np.float64)
        local = unit @ rot.T
        local /= np.linalg.norm(local, axis=1)[:, None]
        y = spherical_harmonics_all(l_top, local)
        phase = np.exp(1j * (kv @ np.asarray(spec.positions[a], dtype=np.float64)))
        f_a, f_b = match_factors(spec, a, columns)
        off = int(offs[a])
        for l in range(l_top + 1):
            pref = (4.0 * np.pi / (np.sqrt(omega) * w[l])) * (1j**l) * phase
            rows = slice(off + l * l, off + (l + 1) ** 2)
            y_rows = np.conj(y[l * l:(l + 1) ** 2])
            a_star[rows] = y_rows * (pref * f_a[l])[None, :]
            b_star[rows] = y_rows * (pref * f_b[l])[None, :]
            udot_norms[rows] = np.asarray(rad.udot_norm)[l]
    return a_star, b_star, udot_norms, offs
