"""Oracle restatement of the special functions on the A/B path (test infrastructure).

Spherical Bessel j_l and j_l' with the reference's three regimes
(`special.py:104-131`): exact limits at x = 0, power series for x < 0.5
(`special.py:49-64`), upward recurrence for x >= l_top (`special.py:67-74`) and
Miller downward recurrence otherwise (`special.py:77-101`).  Spherical
harmonics with Condon-Shortley phase and rows ordered l^2 + l + m
(`special.py:134-179`).  Vectorised over the argument array; each element
follows the same scalar recurrence as the reference.
"""
from __future__ import annotations

import numpy as np


def lm_index(l: int, m: int) -> int:
    """Compound row index l^2 + l + m (`special.py:134-136`)."""
    return l * l + l + m


def _double_factorial(n: int) -> float:
    r = 1.0
    while n > 1:
        r *= n
        n -= 2
    return r


def _series(l_top: int, x: np.ndarray) -> np.ndarray:
    """j_0..j_{l_top}(x) by the power series (`special.py:49-64`)."""
    out = np.zeros((l_top + 1, x.size))
    x2h = 0.5 * x * x
    for l in range(l_top + 1):
        term = x**l / _double_factorial(2 * l + 1)
        total = term.copy()
        active = np.ones(x.size, dtype=bool)
        k = 1
        while active.any():
            term = np.where(active, term * (-x2h / (k * (2 * l + 2 * k + 1))), term)
            total = np.where(active, total + term, total)
            stop = (np.abs(term) <= 1e-18 * np.maximum(np.abs(total), 1e-300)) | (k > 60)
            active &= ~stop
            k += 1
        out[l] = total
    return out


def _upward(l_top: int, x: np.ndarray) -> np.ndarray:
    """Upward recurrence from j_0, j_1 (`special.py:67-74`)."""
    out = np.zeros((l_top + 1, x.size))
    s, c = np.sin(x), np.cos(x)
    out[0] = s / x
    if l_top >= 1:
        out[1] = s / x**2 - c / x
    for l in range(1, l_top):
        out[l + 1] = (2 * l + 1) / x * out[l] - out[l - 1]
    return out


def _downward(l_top: int, x: np.ndarray) -> np.ndarray:
    """Miller downward recurrence normalised on j_0 or j_1 (`special.py:77-101`)."""
    out = np.zeros((l_top + 1, x.size))
    starts = l_top + np.maximum(16, x.astype(np.int64)) + int(2.0 * np.sqrt(l_top + 1))
    for start in np.unique(starts):
        sel = starts == start
        xs = x[sel]
        jp1 = np.zeros(xs.size)
        jl = np.full(xs.size, 1e-30)
        scratch = np.zeros((l_top + 1, xs.size))
        for l in range(int(start), 0, -1):
            jm1 = (2 * l + 1) / xs * jl - jp1
            jp1 = jl
            jl = jm1
            big = np.abs(jl) > 1e250
            if big.any():
                jl = np.where(big, jl * 1e-250, jl)
                jp1 = np.where(big, jp1 * 1e-250, jp1)
                lo = min(l, l_top)
                scratch[lo:] = np.where(big[None, :], scratch[lo:] * 1e-250, scratch[lo:])
            if l - 1 <= l_top:
                scratch[l - 1] = jl
        s, c = np.sin(xs), np.cos(xs)
        j0 = s / xs
        j1 = s / xs**2 - c / xs
        use0 = (np.abs(j0) >= np.abs(j1)) & (scratch[0] != 0)
        if l_top >= 1:
            use1 = ~use0 & (scratch[1] != 0)
            with np.errstate(divide="ignore", invalid="ignore"):
                scale = np.where(use0, j0 / scratch[0],
                                 np.where(use1, j1 / scratch[1], j0 / scratch[0]))
        else:
            scale = j0 / scratch[0]
        out[:, sel] = scratch * scale[None, :]
    return out


def spherical_bessel_all(l_max: int, x) -> tuple[np.ndarray, np.ndarray]:
    """(j_0..j_{l_max}, j'_0..j'_{l_max}) at each x >= 0; shapes (l_max+1, n).

    Regime switch and derivative formula as `special.py:104-131`: orders are
    computed up to l_top = l_max + 1 so j'_{l_max} = j_{l_max-1} - (l_max+1)/x j_{l_max}.
    """
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    if np.any(x < 0):
        raise ValueError("spherical Bessel argument must be >= 0")
    n = l_max + 2
    l_top = n - 1
    j = np.zeros((l_top + 1, x.size))
    zero = x == 0.0
    ser = (x < 0.5) & ~zero
    up = x >= n - 1
    down = ~(zero | ser | up)
    j[0, zero] = 1.0
    if ser.any():
        j[:, ser] = _series(l_top, x[ser])
    if up.any():
        j[:, up] = _upward(l_top, x[up])
    if down.any():
        j[:, down] = _downward(l_top, x[down])
    jp = np.zeros((l_max + 1, x.size))
    nz = ~zero
    jp[0, nz] = -j[1, nz]
    for l in range(1, l_max + 1):
        jp[l, nz] = j[l - 1, nz] - (l + 1) / x[nz] * j[l, nz]
    if l_max >= 1:
        jp[1, zero] = 1.0 / 3.0
    return j[: l_max + 1], jp


def spherical_harmonics_all(l_max: int, directions) -> np.ndarray:
    """Y_lm for l <= l_max on unit directions: ((l_max+1)^2, n) complex.

    Normalised associated Legendre recurrence (sectoral seed, then upward in l)
    times e^{i m phi}; Y_{l,-m} = (-1)^m conj(Y_{l,m}) (`special.py:139-179`).
    """
    d = np.atleast_2d(np.asarray(directions, dtype=np.float64))
    ct = np.clip(d[:, 2], -1.0, 1.0)
    st = np.sqrt(np.maximum(0.0, 1.0 - ct * ct))
    phi = np.arctan2(d[:, 1], d[:, 0])
    npts = d.shape[0]
    p = np.zeros((l_max + 1, l_max + 1, npts))
    p[0, 0] = 1.0 / np.sqrt(4.0 * np.pi)
    for m in range(1, l_max + 1):
        p[m, m] = -np.sqrt((2 * m + 1) / (2.0 * m)) * st * p[m - 1, m - 1]
    for m in range(l_max):
        p[m + 1, m] = np.sqrt(2 * m + 3.0) * ct * p[m, m]
    for m in range(l_max + 1):
        for l in range(m + 2, l_max + 1):
            a = np.sqrt((4.0 * l * l - 1.0) / (l * l - m * m))
            b = np.sqrt(((l - 1.0) ** 2 - m * m) / (4.0 * (l - 1.0) ** 2 - 1.0))
            p[l, m] = a * (ct * p[l - 1, m] - b * p[l - 2, m])
    out = np.zeros(((l_max + 1) ** 2, npts), dtype=np.complex128)
    e1 = np.exp(1j * phi)
    for m in range(l_max + 1):
        e = e1**m
        for l in range(m, l_max + 1):
            y = p[l, m] * e
            out[lm_index(l, m)] = y
            if m:
                out[lm_index(l, -m)] = (-1) ** m * np.conj(y)
    return out


def legendre_all(l_max: int, x) -> np.ndarray:
    """P_0..P_{l_max}(x) by the three-term recurrence (`special.py:22-38`); KAT helper."""
    x = np.clip(np.asarray(x, dtype=np.float64), -1.0, 1.0)
    out = np.zeros((l_max + 1,) + x.shape)
    out[0] = 1.0
    if l_max >= 1:
        out[1] = x
    for l in range(1, l_max):
        out[l + 1] = ((2 * l + 1) * x * out[l] - l * out[l - 1]) / (l + 1)
    return out
