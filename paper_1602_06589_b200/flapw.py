"""FLAPW input types and the GPU matching-coefficient generator.

`RadialBoundaryData` and `SystemSpec` keep the reference fields and validation
(`flapw.py:36-166`).  `compute_AB` (`flapw.py:201-233`) runs the fused sm_100a A/B
generator (`csrc/abgen.cu`) and returns host `StackedCoefficients` in the
reference layout: A*, B* column-major R x N_G windows over capacity-height
allocations, rows per atom ordered l^2 + l + m.
"""
from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .builder import StackedCoefficients
from .errors import ConfigurationError, ContractViolationError
from .matrix import AtomBlockLayout, ComplexDense, DeviceComplexDense

_MIN_WRONSKIAN = 1e-8


_RADIAL_FIELDS = ("u", "u_prime", "udot", "udot_prime", "energy", "udot_norm")


@dataclass
class RadialBoundaryData:
    """One atom's radial solutions at the sphere boundary, one entry per l = 0..l_max: u_l,
    u_l', the energy derivatives and their norms (`flapw.py:36-82`)."""

    u: np.ndarray
    u_prime: np.ndarray
    udot: np.ndarray
    udot_prime: np.ndarray
    energy: np.ndarray
    udot_norm: np.ndarray

    def __post_init__(self):
        for name in _RADIAL_FIELDS:
            setattr(self, name, np.asarray(getattr(self, name), dtype=np.float64))
        want = (len(self.u),)
        odd = [name for name in _RADIAL_FIELDS if getattr(self, name).shape != want]
        if odd:
            raise ContractViolationError(f"radial arrays {odd} do not have the {want[0]} entries of u")
        if (self.udot_norm < 0).any():
            raise ContractViolationError("a norm of udot cannot be negative")
        # the match factors divide by the Wronskian W_l = udot_l u_l' - u_l udot_l'
        if (np.abs(self.wronskian) < _MIN_WRONSKIAN).any():
            raise ContractViolationError(
                f"radial pair (u, udot) nearly dependent: a |Wronskian| is under {_MIN_WRONSKIAN}")

    @property
    def wronskian(self) -> np.ndarray:
        return self.udot * self.u_prime - self.u * self.udot_prime

    @property
    def l_max(self) -> int:
        return len(self.u) - 1

    def to_json_dict(self) -> dict:
        return {name: getattr(self, name).tolist() for name in _RADIAL_FIELDS}

    @classmethod
    def from_json_dict(cls, d: dict) -> "RadialBoundaryData":
        return cls(**{name: np.asarray(vals, dtype=np.float64) for name, vals in d.items()})


_SPEC_ARRAYS = (("positions", np.float64), ("rotations", np.float64), ("mt_radius", np.float64),
                ("l_sph", np.int64), ("l_nonsph", np.int64), ("k_point", np.float64),
                ("k_vectors", np.float64))


def _proper_or_improper_rotation(r: np.ndarray) -> str | None:
    """None for an orthogonal 3x3 matrix of determinant +-1 (tolerance 1e-12), else what fails."""
    if np.abs(r.T @ r - np.eye(3)).max() > 1e-12:
        return "is not orthogonal"
    if abs(abs(np.linalg.det(r)) - 1.0) > 1e-12:
        return "has a determinant of modulus other than one"
    return None


@dataclass
class SystemSpec:
    """Everything `compute_AB` needs for one k-point: atoms (positions, local frames, sphere
    radii, cutoffs, radial data), the K = k + G vectors and the cell volume (`flapw.py:85-166`)."""

    positions: np.ndarray
    rotations: np.ndarray
    mt_radius: np.ndarray
    l_sph: np.ndarray
    l_nonsph: np.ndarray
    k_point: np.ndarray
    k_vectors: np.ndarray
    omega: float
    radial: list

    def __post_init__(self):
        for name, kind in _SPEC_ARRAYS:
            setattr(self, name, np.asarray(getattr(self, name), dtype=kind))
        atoms = self.n_atoms
        kv = self.k_vectors
        if kv.ndim != 2 or kv.shape[1] != 3 or kv.shape[0] == 0:
            raise ContractViolationError("k_vectors is a non-empty list of 3-vectors")
        if self.omega <= 0:
            raise ContractViolationError("the cell volume omega is positive")
        if (self.l_nonsph > self.l_sph).any():
            raise ConfigurationError("l_nonsph is capped by l_sph, atom by atom")
        if (self.mt_radius <= 0).any():
            raise ContractViolationError("every muffin-tin radius is positive")
        if self.rotations.shape != (atoms, 3, 3):
            raise ContractViolationError(f"rotations holds a 3x3 matrix for each of the {atoms} atoms")
        for a, frame in enumerate(self.rotations):
            fault = _proper_or_improper_rotation(frame)
            if fault:
                raise ContractViolationError(f"local frame of atom {a} {fault}")
        if len(self.radial) != atoms:
            raise ContractViolationError(f"radial holds one entry for each of the {atoms} atoms")
        short = [a for a, rad in enumerate(self.radial) if rad.l_max < self.l_sph[a]]
        if short:
            raise ContractViolationError(f"radial data of atoms {short} ends before their l_sph")

    @property
    def n_atoms(self) -> int:
        return self.positions.shape[0]

    @property
    def n_basis(self) -> int:
        return self.k_vectors.shape[0]

    def layout(self) -> AtomBlockLayout:
        heights = tuple(int((l + 1) ** 2) for l in self.l_sph)
        return AtomBlockLayout(heights, int((self.l_sph.max() + 1) ** 2))

    def to_json_dict(self) -> dict:
        doc = {name: getattr(self, name).tolist() for name, _ in _SPEC_ARRAYS}
        doc["omega"] = self.omega
        doc["radial"] = [rad.to_json_dict() for rad in self.radial]
        return doc

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict(), sort_keys=True)

    @classmethod
    def from_json_dict(cls, d: dict) -> "SystemSpec":
        d = dict(d)
        d["radial"] = [RadialBoundaryData.from_json_dict(r) for r in d["radial"]]
        return cls(**d)

    @classmethod
    def from_json(cls, text: str) -> "SystemSpec":
        return cls.from_json_dict(json.loads(text))


def compute_AB(spec: SystemSpec) -> StackedCoefficients:
    """Matching coefficients A*, B* and row norms, generated on the GPU (`flapw.py:201-233`).

    The stacks stay in HBM (`DeviceComplexDense`): `build_all` uses them in place (or, while
    they are untouched, builds from the spec itself on the device pipeline), and the first host
    access downloads them into pinned memory with the reference's capacity-height layout
    (`flapw.py:209-212`), one contiguous DMA per stack."""
    from . import device
    from .pipeline import DeviceSpec, ab_generate_device

    device.require_cuda()
    layout = spec.layout()
    dspec = DeviceSpec(spec)
    n = spec.n_basis
    # Generated with the host allocation's leading dimension (capacity rows, flapw.py:209-212).
    cap = layout.capacity_rows
    a_dev = device.empty_matrix(cap, n, cap, zero=True)
    b_dev = device.empty_matrix(cap, n, cap, zero=True)
    ab_generate_device(dspec, a_dev, b_dev, None, cap, None)
    # per-row ||udot|| (flapw.py:232) straight from the radial data: no device round trip, so
    # the call returns while the generator still runs
    norms = np.array(dspec.udot_rows, dtype=np.float64)
    coeffs = StackedCoefficients(DeviceComplexDense(a_dev, cap, n, layout.total_rows),
                                 DeviceComplexDense(b_dev, cap, n, layout.total_rows), layout, norms)
    # the device copy of the spec these stacks are a function of: build_all runs from it while
    # the stacks stay untouched (builder._build_from_origin)
    coeffs._origin = dspec
    coeffs._origin_stacks = (coeffs.A_star, coeffs.B_star)  # these very objects, not replacements
    return coeffs


def match_factors(spec: SystemSpec, atom: int):
    """Real radial match factors (f_A, f_B), each (l_sph+1, N_G), of one atom on the GPU
    (`flapw.py:179-198`; `hsdla_match_factors`, same Bessel code as `compute_AB`)."""
    import ctypes

    from . import _native, device
    from .pipeline import DeviceSpec

    t = device.require_cuda()
    if not 0 <= atom < spec.n_atoms:
        raise ContractViolationError(f"atom index {atom} out of range")
    ds = DeviceSpec(spec)
    n = ds.n_basis
    l_top = ds.l_sph.astype(np.int32)
    f_row = np.concatenate(([0], np.cumsum(l_top.astype(np.int64) + 1)[:-1])).astype(np.int64)
    rows = int((l_top + 1).sum())
    fa = t.empty((rows, max(n, 1)), dtype=t.float64, device="cuda")
    fb = t.empty((rows, max(n, 1)), dtype=t.float64, device="cuda")
    args = _native.AbArgs()
    args.n_atoms, args.n_basis = ds.n_atoms, n
    args.k_vectors, args.positions = ds.kv.data_ptr(), ds.pos.data_ptr()
    args.rotations, args.mt_radius = ds.rot.data_ptr(), ds.rmt.data_ptr()
    args.radial, args.radial_stride = ds.radial.data_ptr(), ds.radial_stride
    args.l_sph = l_top.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    args.omega = ds.omega
    _native.check(_native.load().hsdla_match_factors(
        device.ctx(), ctypes.byref(args), f_row.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        device.ptr(fa), device.ptr(fb), max(n, 1)), "hsdla_match_factors")
    r0, r1 = int(f_row[atom]), int(f_row[atom]) + int(l_top[atom]) + 1
    return fa[r0:r1, :n].cpu().numpy(), fb[r0:r1, :n].cpu().numpy()


# ---- input side: Gaunt-sum assembly of the coupling matrices ----------

BB_DIAG_NORM_POWER = 1  # flapw.py:31


@dataclass
class RadialIntegrals:
    """Radial integrals of one atom's coupling-matrix assembly (`flapw.py:253-273`): arrays
    indexed (l', l, L'') with the compound potential index L'' = (l'', m'') up to l_nonsph;
    uu / dd satisfy c[l', l, (l'', m'')] = (-1)^m'' conj(c[l, l', (l'', -m'')]) and du is that
    partner of ud, so the assembled T_AA / T_BB are Hermitian and T_BA = T_AB^H."""

    c_uu: np.ndarray
    c_dd: np.ndarray
    c_ud: np.ndarray
    c_du: np.ndarray

    @property
    def l_nonsph(self) -> int:
        return self.c_uu.shape[0] - 1


def _pairing(c: np.ndarray) -> np.ndarray:
    """The Hermitian-compatibility involution on (l', l, L'') arrays (`flapw.py:276-286`):
    swap l' <-> l, conjugate, and map L'' = (l'', m'') to (-1)^m'' x entry (l'', -m'')."""
    l_pot = int(round(np.sqrt(c.shape[2]))) - 1
    lm = np.array([(l, m) for l in range(l_pot + 1) for m in range(-l, l + 1)], dtype=np.int64)
    flipped = lm[:, 0] * (lm[:, 0] + 1) - lm[:, 1]  # compound index of (l'', -m'')
    parity = np.where(lm[:, 1] % 2 == 0, 1.0, -1.0)
    return np.conj(np.swapaxes(c, 0, 1))[:, :, flipped] * parity


def synth_radial_integrals(seed: int, l_nonsph: int, scale: float = 0.5) -> RadialIntegrals:
    """Seeded radial integrals satisfying the pairing (`flapw.py:289-307`; the same normal
    draws in the same order, so a seed gives the reference's integrals)."""
    gen = np.random.default_rng(seed)
    shape = (l_nonsph + 1, l_nonsph + 1, (l_nonsph + 1) ** 2)
    z = [gen.standard_normal((2,) + shape) for _ in range(3)]  # (re, im) of uu, dd, ud
    x_uu, x_dd, c_ud = (scale * (v[0] + 1j * v[1]) for v in z)
    return RadialIntegrals(c_uu=0.5 * (x_uu + _pairing(x_uu)), c_dd=0.5 * (x_dd + _pairing(x_dd)),
                           c_ud=c_ud, c_du=_pairing(c_ud))


def assemble_T(spec: SystemSpec, radial_integrals: list):
    """Per-atom coupling matrices from Gaunt sums plus diagonal terms (`flapw.py:310-363`):
    the dense (l_nonsph+1)^2 block is sum_k c[l(p), l(q), k] G[p, q, k] (G = the Gaunt tensor,
    computed on the GPU over the reference's quadrature grid), the diagonal carries the energy
    parameters (AA), energy x ||udot|| (BB) and ones (AB); T_BA is never built.  The result has
    the dense-block + diagonal-tail shape the build's T-structure split uses."""
    from .builder import TMatrixSet
    from . import _native, device
    from .special import _gaunt_device

    if len(radial_integrals) != spec.n_atoms:
        raise ContractViolationError("need radial integrals per atom")
    t = device.require_cuda()
    lib = _native.load()
    t_aa, t_ab, t_bb = [], [], []
    g_cache = {}
    for a in range(spec.n_atoms):
        ri = radial_integrals[a]
        l_n, l_s = int(spec.l_nonsph[a]), int(spec.l_sph[a])
        if ri.l_nonsph != l_n:
            raise ContractViolationError(
                f"atom {a}: integrals cover l_nonsph={ri.l_nonsph}, spec says {l_n}")
        for name, c in (("uu", ri.c_uu), ("dd", ri.c_dd)):
            if np.max(np.abs(c - _pairing(c))) > 1e-12:
                raise ContractViolationError(f"atom {a}: {name} integrals violate the Hermitian pairing")
        if np.max(np.abs(ri.c_du - _pairing(ri.c_ud))) > 1e-12:
            raise ContractViolationError(f"atom {a}: du integrals are not the conjugate partner of ud")
        if l_n not in g_cache:
            g_cache[l_n] = _gaunt_device(l_n, l_n)
        g = g_cache[l_n]
        n_l, n_full = l_n + 1, (l_s + 1) ** 2
        n_pot = n_l * n_l
        rad = spec.radial[a]
        e = np.asarray(rad.energy, dtype=np.float64)[:l_s + 1]
        e_bb = e * np.asarray(rad.udot_norm, dtype=np.float64)[:l_s + 1] ** BB_DIAG_NORM_POWER
        outs = []
        for c, diag, unit in ((ri.c_uu, e, 0.0), (ri.c_ud, None, 1.0), (ri.c_dd, e_bb, 0.0)):
            cd = t.from_numpy(np.ascontiguousarray(c, dtype=np.complex128)).cuda()
            dd = t.from_numpy(np.ascontiguousarray(diag)).cuda() if diag is not None else None
            out = t.empty((n_full, n_full), dtype=t.complex128, device="cuda")
            _native.check(lib.hsdla_gaunt_sum(device.ctx(), n_full, n_l, n_pot, device.ptr(cd),
                                              device.ptr(g), device.ptr(dd) if dd is not None
                                              else None, unit, device.ptr(out)), "hsdla_gaunt_sum")
            outs.append(ComplexDense(out.cpu().numpy().T))  # (col, row) storage -> F-order
        t_aa.append(outs[0])
        t_ab.append(outs[1])
        t_bb.append(outs[2])
    return TMatrixSet(t_aa=t_aa, t_ab=t_ab, t_bb=t_bb, l_sph=[int(x) for x in spec.l_sph],
                      l_nonsph=[int(x) for x in spec.l_nonsph])
