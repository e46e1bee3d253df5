"""Oracle restatement of the input-side Gaunt machinery (test infrastructure only).

* `gaunt_tensor` — G[L', L, L''] = sum_pts w conj(Y_L') Y_L Y_L'' over the product grid of
  Gauss-Legendre nodes in cos(theta) (2 l_max + 1 of them) times uniform phi (4 l_max + 1),
  exact for triple products up to l_max (`special.py:189-204`, `:227-244`);
* `assemble_T` — per atom, the dense (l_nonsph+1)^2 block sum_k c[l(p), l(q), k] G[p, q, k]
  of the uu / ud / dd integrals, plus energy (AA), energy x ||udot|| (BB) and 1 (AB) on the
  full diagonal (`flapw.py:310-363`).

Pinned by tests/test_oracle_golden.py against tests/golden/assemble_t.npz (the reference's own
outputs, tests/golden/make_golden_assemble.py).
"""
from __future__ import annotations

import numpy as np

from .special import spherical_harmonics_all


def quadrature_grid(l_max: int, refine: int = 1):
    """(Y on the grid, weights) (`special.py:189-204`)."""
    nodes, node_w = np.polynomial.legendre.leggauss(refine * (2 * l_max + 1))
    n_az = refine * (4 * l_max + 1)
    az = 2.0 * np.pi * np.arange(n_az) / n_az
    grid_c, grid_a = np.meshgrid(nodes, az, indexing="ij")
    w = (node_w[:, None] * np.full((1, n_az), 2.0 * np.pi / n_az)).ravel()
    c, a = grid_c.ravel(), grid_a.ravel()
    s = np.sqrt(np.clip(1.0 - c * c, 0.0, None))
    dirs = np.column_stack((s * np.cos(a), s * np.sin(a), c))
    return spherical_harmonics_all(l_max, dirs), w


def gaunt_tensor(l_row_max: int, l_pot_max: int, refine: int = 1) -> np.ndarray:
    """(n_row, n_row, n_pot) Gaunt tensor (`special.py:227-244`)."""
    y, w = quadrature_grid(max(l_row_max, l_pot_max), refine)
    n_row, n_pot = (l_row_max + 1) ** 2, (l_pot_max + 1) ** 2
    yr, yp = y[:n_row], y[:n_pot]
    return np.einsum("ip,jp,kp->ijk", np.conj(yr) * w, yr, yp)


def assemble_T(l_sph, l_nonsph, energies, udot_norms, integrals):
    """Lists (t_aa, t_ab, t_bb) of per-atom dense arrays (`flapw.py:310-363`);
    `integrals[a]` = (c_uu, c_ud, c_dd)."""
    t_aa, t_ab, t_bb = [], [], []
    for a, (ls, ln) in enumerate(zip(l_sph, l_nonsph)):
        n_dense, n_full = (ln + 1) ** 2, (ls + 1) ** 2
        g = gaunt_tensor(ln, ln)
        l_of = np.array([l for l in range(ln + 1) for _ in range(2 * l + 1)])
        diag_l = np.array([l for l in range(ls + 1) for _ in range(2 * l + 1)])
        idx = np.arange(n_full)
        blocks = []
        for c in integrals[a]:
            m = np.zeros((n_full, n_full), dtype=np.complex128)
            m[:n_dense, :n_dense] = np.einsum("pqk,pqk->pq", c[np.ix_(l_of, l_of)], g)
            blocks.append(m)
        aa, ab, bb = blocks
        aa[idx, idx] += energies[a][diag_l]
        bb[idx, idx] += energies[a][diag_l] * udot_norms[a][diag_l]
        ab[idx, idx] += 1.0
        t_aa.append(aa)
        t_ab.append(ab)
        t_bb.append(bb)
    return t_aa, t_ab, t_bb
