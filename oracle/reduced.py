"""Oracle restatement of the Legendre-reduced A-side overlap (test infrastructure).

`reduced_s_aa(f, wronskians, positions, k_vectors, omega)` follows reference
`oracle.py:186-216` (reduced_S_AA); `reduced_inputs(spec)` follows `flapw.py:236-250`
(reduced_overlap_inputs) with `match_factors` (`flapw.py:179-198`).  Plain numpy.
"""
from __future__ import annotations

import numpy as np

from .flapw import match_factors, wronskian
from .special import legendre_all


def reduced_inputs(spec):
    """(f per atom (l+1, N_G), W per atom (l+1,)) of `flapw.py:236-250`."""
    f, w = [], []
    for a in range(spec.n_atoms):
        f_a, _ = match_factors(spec, a)
        f.append(f_a)
        w.append(wronskian(spec.radial[a])[: int(spec.l_sph[a]) + 1])
    return f, w


def reduced_s_aa(f, wronskians, positions, k_vectors, omega) -> np.ndarray:
    """Full N_G x N_G reduced A-side overlap (`oracle.py:186-216`)."""
    k = np.asarray(k_vectors, dtype=np.float64)
    norms = np.linalg.norm(k, axis=1)
    nz = norms > 0
    unit = np.zeros_like(k)
    unit[nz] = k[nz] / norms[nz, None]
    cos = np.clip(unit @ unit.T, -1.0, 1.0)
    cos[~nz, :] = 1.0          # a zero K-vector is parallel to everything
    cos[:, ~nz] = 1.0
    leg = legendre_all(max(fa.shape[0] - 1 for fa in f), cos)
    n = k.shape[0]
    out = np.zeros((n, n), dtype=np.complex128)
    for x_a, f_a, w_a in zip(np.asarray(positions, dtype=np.float64), f, wronskians):
        ph = np.exp(1j * (k @ x_a))
        radial = np.zeros((n, n))
        for l in range(f_a.shape[0]):
            radial += (2 * l + 1) / (4.0 * np.pi) / (w_a[l] ** 2) * np.outer(f_a[l], f_a[l]) * leg[l]
        out += (np.conj(ph)[:, None] * ph[None, :]) * radial
    out *= (4.0 * np.pi) ** 2 / omega
    return out
