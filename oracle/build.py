"""Oracle restatement of the HSDLA build (test infrastructure).

`build_all` restates reference `builder.py:403-474` with the phases
`build_H_ABBA_BB` (`builder.py:212-248`), `build_S` (`builder.py:199-209`) and
`build_H_AA` (`builder.py:251-315`) on the same BLAS/LAPACK routines the
reference's "optimized" backend calls (`kernels.py:237-272`: zherk, zher2k,
zgemm, zhemm, ztrmm, zpotrf through scipy), plus the mirror
(`matrix.py:216-226`).  `naive_S`/`naive_H` are independent dense-numpy
restatements of the entrywise oracle formulas (`oracle.py:23-124`), and
`predict_flops`/`estimate_memory` restate the integer closed forms
(`builder.py:318-370`).  Inputs are plain numpy arrays.
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import blas as _blas
from scipy.linalg import lapack as _lapack

LEDGER_KINDS = ("hermitian_rank_k", "hermitian_rank_2k", "general_product",
                "hermitian_product", "triangular_product", "cholesky", "row_scale")


def cholesky_flops(n: int) -> int:
    """4 n^3 // 3 (`matrix.py:197-199`)."""
    return 4 * n**3 // 3


def new_ledger() -> dict:
    return {k: 0 for k in LEDGER_KINDS}


def hermitian_full(t_lower: np.ndarray) -> np.ndarray:
    """Full Hermitian matrix from the lower triangle, real diagonal (`kernels.py:197-201`)."""
    full = np.tril(t_lower) + np.tril(t_lower, -1).conj().T
    np.fill_diagonal(full, full.diagonal().real)
    return full


def potrf_lower(t: np.ndarray):
    """(factor, pivot): Cholesky of tril(t); pivot = -1 on success (`kernels.py:119-132`, `:266-272`)."""
    lower = np.tril(t)
    if np.isnan(lower).any():
        raise ValueError("NaN in Cholesky input (lower triangle)")
    factor, info = _lapack.zpotrf(np.asfortranarray(lower), lower=1, clean=1, overwrite_a=0)
    if info > 0:
        return None, info - 1
    if info < 0:
        raise ValueError(f"zpotrf rejected argument {-info}")
    return factor, -1


def mirror_lower(c: np.ndarray) -> np.ndarray:
    """Upper <- conj(lower^T), diagonal imag <- 0 (`matrix.py:216-226`)."""
    n = c.shape[0]
    out = np.tril(c, -1)
    out = out + out.conj().T
    out[np.arange(n), np.arange(n)] = c.diagonal().real
    return out


def build_all(a, b, udot_norms, heights, t_aa, t_ab, t_bb, force_general_path=False):
    """(H, S, ledger, hpd_mask) as reference build_all with backup=True.

    `a`, `b`: (R, N) complex; `heights`: per-atom block heights; `t_*`:
    per-atom m x m arrays (m <= height).  The inputs are not modified.
    """
    a = np.asfortranarray(np.array(a, dtype=np.complex128))
    b = np.asfortranarray(np.array(b, dtype=np.complex128))
    r, n = a.shape
    offs = np.concatenate(([0], np.cumsum(heights))).astype(np.int64)
    led = new_ledger()
    sizes = [int(t.shape[0]) for t in t_aa]

    # H_ABBA_BB: Z_a = T_AB^H A_a + 1/2 T_BB B_a, compacted, then one ZHER2K (builder.py:227-247)
    h = np.zeros((n, n), dtype=np.complex128, order="F")
    zs, bs = [], []
    for at, m in enumerate(sizes):
        off = int(offs[at])
        a_blk = a[off:off + m]
        b_blk = b[off:off + m]
        z = _blas.zgemm(1.0, np.asfortranarray(t_ab[at]), a_blk, trans_a=2)
        z = _blas.zhemm(0.5, np.asfortranarray(t_bb[at]), b_blk, beta=1.0, c=z, side=0, lower=1)
        led["general_product"] += 8 * m * n * m
        led["hermitian_product"] += 8 * m * m * n
        zs.append(z)
        bs.append(b_blk)
    zstar = np.asfortranarray(np.vstack(zs)) if zs else np.zeros((0, n), complex, order="F")
    bstar = np.asfortranarray(np.vstack(bs)) if bs else np.zeros((0, n), complex, order="F")
    if zstar.shape[0] and n:
        h = _blas.zher2k(1.0, zstar, bstar, beta=1.0, c=h, trans=2, lower=1, overwrite_c=1)
    led["hermitian_rank_2k"] += 8 * zstar.shape[0] * n * n

    # S: ZHERK(A), scale B rows by ||udot||, ZHERK(B) (builder.py:199-209)
    s = np.zeros((n, n), dtype=np.complex128, order="F")
    if r and n:
        s = _blas.zherk(1.0, a, beta=1.0, c=s, trans=2, lower=1, overwrite_c=1)
    led["hermitian_rank_k"] += 4 * r * n * n
    bsc = np.asfortranarray(b * np.asarray(udot_norms, dtype=np.float64)[:, None])
    led["row_scale"] += 2 * r * n
    if r and n:
        s = _blas.zherk(1.0, bsc, beta=1.0, c=s, trans=2, lower=1, overwrite_c=1)
    led["hermitian_rank_k"] += 4 * r * n * n

    # H_AA: per-atom Cholesky dispatch (builder.py:274-315)
    ys, xs, anots, mask = [], [], [], []
    for at, m in enumerate(sizes):
        off = int(offs[at])
        a_blk = a[off:off + m]
        fac = None
        if not force_general_path:
            fac, piv = potrf_lower(t_aa[at])
            if fac is not None:
                led["cholesky"] += cholesky_flops(m)
        if fac is None:
            x = _blas.zhemm(1.0, np.asfortranarray(t_aa[at]), a_blk, side=0, lower=1)
            led["hermitian_product"] += 8 * m * m * n
            xs.append(x)
            anots.append(a_blk)
            mask.append(False)
        else:
            y = _blas.ztrmm(1.0, fac, np.array(a_blk, order="F"), side=0, lower=1, trans_a=2, diag=0)
            led["triangular_product"] += 4 * m * m * n
            # the reference stacks Y from the bottom of the scratch buffer: last atom on top
            ys.insert(0, y)
            mask.append(True)
    if xs:
        xst = np.asfortranarray(np.vstack(xs))
        ast = np.asfortranarray(np.vstack(anots))
        h = _blas.zgemm(1.0, ast, xst, beta=1.0, c=h, trans_a=2, overwrite_c=1)
        led["general_product"] += 8 * n * n * xst.shape[0]
    if ys:
        yst = np.asfortranarray(np.vstack(ys))
        h = _blas.zherk(1.0, yst, beta=1.0, c=h, trans=2, lower=1, overwrite_c=1)
        led["hermitian_rank_k"] += 4 * yst.shape[0] * n * n
    return mirror_lower(h), mirror_lower(s), led, mask


def naive_S(a, b, udot_norms) -> np.ndarray:
    """Full S = A^H A + B^H diag(||udot||^2) B (`oracle.py:23-36`, `:75-87`)."""
    w2 = np.asarray(udot_norms, dtype=np.float64) ** 2
    return a.conj().T @ a + b.conj().T @ (w2[:, None] * b)


def naive_H(a, b, heights, t_aa, t_ab, t_bb) -> np.ndarray:
    """Full H = sum_a A_a^H W1_a + B_a^H W2_a with W1 = T_AA A + T_AB B,
    W2 = T_AB^H A + T_BB B, T used as stored (`oracle.py:38-72`, `:105-124`)."""
    n = a.shape[1]
    offs = np.concatenate(([0], np.cumsum(heights))).astype(np.int64)
    h = np.zeros((n, n), dtype=np.complex128)
    for at, t in enumerate(t_aa):
        m = t.shape[0]
        off = int(offs[at])
        aa, bb = a[off:off + m], b[off:off + m]
        w1 = t_aa[at] @ aa + t_ab[at] @ bb
        w2 = t_ab[at].conj().T @ aa + t_bb[at] @ bb
        h += aa.conj().T @ w1 + bb.conj().T @ w2
    return h


def h_matvec(a, b, heights, t_aa, t_ab, t_bb, v) -> np.ndarray:
    """H @ v in O(R N) without forming H (full-size parity projections).

    Uses the Hermitian forms of T_AA / T_BB built from their lower triangles,
    which is what every build path reads (`kernels.py:197-201`)."""
    offs = np.concatenate(([0], np.cumsum(heights))).astype(np.int64)
    out = np.zeros((a.shape[1],) + v.shape[1:], dtype=np.complex128)
    for at, t in enumerate(t_aa):
        m = t.shape[0]
        off = int(offs[at])
        aa, bb = a[off:off + m], b[off:off + m]
        av, bv = aa @ v, bb @ v
        taa, tbb, tab = hermitian_full(t_aa[at]), hermitian_full(t_bb[at]), t_ab[at]
        w1 = taa @ av + tab @ bv
        w2 = tab.conj().T @ av + tbb @ bv
        out += aa.conj().T @ w1 + bb.conj().T @ w2
    return out


def s_matvec(a, b, udot_norms, v) -> np.ndarray:
    """S @ v in O(R N)."""
    w2 = np.asarray(udot_norms, dtype=np.float64) ** 2
    v2 = v if v.ndim == 2 else v[:, None]
    out = a.conj().T @ (a @ v2) + b.conj().T @ (w2[:, None] * (b @ v2))
    return out if v.ndim == 2 else out[:, 0]


def predict_flops(heights, n_g: int, hpd_mask) -> dict:
    """Closed-form ledger of one composed build (`builder.py:336-370`)."""
    heights = [int(h) for h in heights]
    mask = [bool(x) for x in hpd_mask]
    led = new_ledger()
    r = sum(heights)
    ng2 = n_g * n_g
    led["hermitian_rank_k"] += 8 * r * ng2
    led["row_scale"] += 2 * r * n_g
    for h in heights:
        led["general_product"] += 8 * h * h * n_g
        led["hermitian_product"] += 8 * h * h * n_g
    led["hermitian_rank_2k"] += 8 * r * ng2
    r_hpd = sum(h for h, m in zip(heights, mask) if m)
    for h, m in zip(heights, mask):
        if m:
            led["cholesky"] += cholesky_flops(h)
            led["triangular_product"] += 4 * h * h * n_g
        else:
            led["hermitian_product"] += 8 * h * h * n_g
    led["general_product"] += 8 * (r - r_hpd) * ng2
    led["hermitian_rank_k"] += 4 * r_hpd * ng2
    return led


def estimate_memory(n_atoms: int, n_l: int, n_g: int, backup: bool) -> int:
    """Peak bytes closed form (`builder.py:318-333`)."""
    stacks = 32 * n_atoms * n_l * n_g
    total = stacks + 32 * n_g * n_g
    if backup:
        total += max(stacks - 16 * n_g * n_g, 0)
    return total


def rel_fro(x, y) -> float:
    """||X - Y||_F / max(||Y||_F, tiny) (`oracle.py:143-156`)."""
    return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), np.finfo(np.float64).tiny))
