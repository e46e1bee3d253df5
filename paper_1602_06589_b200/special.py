"""Special functions of the A/B generation on the GPU (drop-in for reference `special.py`).

`spherical_bessel_all` (`special.py:104-131`) and `spherical_harmonics_all`
(`special.py:139-179`) run the same device code as the A/B generator (`csrc/abgen.cu`,
`csrc/bessel.cuh`): the three Bessel regimes and the normalised-Legendre recurrence with the
reference's rounding sequence.  Both accept many points per call (one kernel launch);
scalar calls keep the reference's return shapes.  Orders up to HSDLA_MAX_LSPH (14).
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

from . import _native, device
from .errors import ContractViolationError


def lm_index(l: int, m: int) -> int:
    """Row index of (l, m) in the compound ordering l^2 + l + m (`special.py:134-136`)."""
    return l * l + l + m


def _check_l(l_max: int) -> None:
    if l_max < 0 or l_max > _native.MAX_LSPH:
        raise ContractViolationError(f"l_max must lie in [0, {_native.MAX_LSPH}], got {l_max}")


def spherical_bessel_all(l_max: int, x):
    """j_0..j_{l_max}(x) and j'_0..j'_{l_max}(x) for x >= 0 (`special.py:104-131`).

    Scalar x: two arrays of length l_max + 1 (the reference's return).  Array x: two
    (l_max + 1, len(x)) arrays, column i for x[i]."""
    _check_l(l_max)
    scalar = np.ndim(x) == 0
    xs = np.atleast_1d(np.asarray(x, dtype=np.float64)).ravel()
    if np.any(xs < 0) or np.any(np.isnan(xs)):
        raise ContractViolationError("spherical Bessel argument must be >= 0")
    t = device.require_cuda()
    n = xs.size
    xd = t.from_numpy(np.ascontiguousarray(xs)).cuda()
    j = t.empty((l_max + 1, max(n, 1)), dtype=t.float64, device="cuda")
    jp = t.empty((l_max + 1, max(n, 1)), dtype=t.float64, device="cuda")
    _native.check(_native.load().hsdla_spherical_bessel(device.ctx(), l_max, n, device.ptr(xd),
                                                        device.ptr(j), device.ptr(jp)),
                  "hsdla_spherical_bessel")
    j, jp = j[:, :n].cpu().numpy(), jp[:, :n].cpu().numpy()
    if scalar:
        return j[:, 0].copy(), jp[:, 0].copy()
    return j, jp


def spherical_harmonics_all(l_max: int, directions) -> np.ndarray:
    """All Y_lm up to l_max at unit direction(s): ((l_max+1)^2, npts) complex, rows
    l^2 + l + m, Condon-Shortley phase (`special.py:139-179`)."""
    _check_l(l_max)
    d = np.atleast_2d(np.asarray(directions, dtype=np.float64))
    if d.shape[1] != 3:
        raise ContractViolationError("directions must be 3-vectors")
    if np.any(np.abs(np.linalg.norm(d, axis=1) - 1.0) > 1e-10):
        raise ContractViolationError("directions must be unit vectors")
    t = device.require_cuda()
    n = d.shape[0]
    dd = t.from_numpy(np.ascontiguousarray(d)).cuda()
    y = t.empty(((l_max + 1) ** 2, max(n, 1)), dtype=t.complex128, device="cuda")
    _native.check(_native.load().hsdla_spherical_harmonics(device.ctx(), l_max, n, device.ptr(dd),
                                                           device.ptr(y)),
                  "hsdla_spherical_harmonics")
    return y[:, :n].cpu().numpy()


def spherical_harmonic(l: int, m: int, direction) -> complex:
    """Single Y_lm at one unit direction (`special.py:182-186`)."""
    if l < 0 or abs(m) > l:
        raise ContractViolationError(f"invalid (l, m) = ({l}, {m})")
    return complex(spherical_harmonics_all(l, direction)[lm_index(l, m), 0])


GAUNT_L_MAX = 12  # special.py:19


@lru_cache(maxsize=8)
def _quadrature_grid(l_max: int, refine: int = 1):
    """Product grid exact for triple products of harmonics up to l_max (`special.py:189-204`):
    Gauss-Legendre in cos(theta) x uniform phi; returns device Y ((l_max+1)^2 x npts) and
    device weights.  The nodes are constants computed once on the host."""
    t = device.require_cuda()
    cos_t, w_t = np.polynomial.legendre.leggauss(refine * (2 * l_max + 1))
    n_phi = refine * (4 * l_max + 1)
    ang = np.linspace(0.0, 2.0 * np.pi, n_phi, endpoint=False)
    ct, ph = (g.ravel() for g in np.meshgrid(cos_t, ang, indexing="ij"))
    w = np.outer(w_t, np.full(n_phi, 2.0 * np.pi / n_phi)).ravel()
    sin_t = np.sqrt(np.clip(1.0 - ct * ct, 0.0, None))
    dirs = np.column_stack((sin_t * np.cos(ph), sin_t * np.sin(ph), ct))
    n = dirs.shape[0]
    dd = t.from_numpy(np.ascontiguousarray(dirs)).cuda()
    y = t.empty(((l_max + 1) ** 2, n), dtype=t.complex128, device="cuda")
    _native.check(_native.load().hsdla_spherical_harmonics(device.ctx(), l_max, n, device.ptr(dd),
                                                           device.ptr(y)),
                  "hsdla_spherical_harmonics")
    return y, t.from_numpy(w).cuda()


def _gaunt_device(l_row_max: int, l_pot_max: int, refine: int = 1):
    l_max = max(l_row_max, l_pot_max)
    if l_max > GAUNT_L_MAX:
        raise ContractViolationError(f"gaunt supports l <= {GAUNT_L_MAX}")
    t = device.require_cuda()
    y, w = _quadrature_grid(l_max, refine)
    n_row, n_pot = (l_row_max + 1) ** 2, (l_pot_max + 1) ** 2
    g = t.empty((n_row, n_row, n_pot), dtype=t.complex128, device="cuda")
    _native.check(_native.load().hsdla_gaunt_tensor(device.ctx(), n_row, n_pot, y.shape[1],
                                                    y.shape[1], device.ptr(y), device.ptr(w),
                                                    device.ptr(g)), "hsdla_gaunt_tensor")
    return g


def gaunt_tensor(l_row_max: int, l_pot_max: int) -> np.ndarray:
    """G[L', L, L''] = gaunt(L', L, L'') for all compound indices in range, shape
    ((l_row_max+1)^2, (l_row_max+1)^2, (l_pot_max+1)^2) (`special.py:227-244`), on the GPU."""
    return _gaunt_device(l_row_max, l_pot_max).cpu().numpy()


def gaunt(lp_mp, l_m, lpp_mpp, refine: int = 1) -> complex:
    """Integral of conj(Y_{l',m'}) Y_{l,m} Y_{l'',m''} over the unit sphere (`special.py:207-224`);
    `refine` multiplies the quadrature resolution."""
    lp, mp = lp_mp
    l, m = l_m
    lpp, mpp = lpp_mpp
    l_max = max(lp, l, lpp)
    if l_max > GAUNT_L_MAX:
        raise ContractViolationError(f"gaunt supports l <= {GAUNT_L_MAX}")
    for ll, mm in ((lp, mp), (l, m), (lpp, mpp)):
        if ll < 0 or abs(mm) > ll:
            raise ContractViolationError(f"invalid (l, m) = ({ll}, {mm})")
    g = _gaunt_device(l_max, l_max, refine)
    return complex(g[lm_index(lp, mp), lm_index(l, m), lm_index(lpp, mpp)].item())
