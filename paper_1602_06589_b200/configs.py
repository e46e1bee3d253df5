"""Seeded synthetic systems for the BASELINE.json configurations C1-C5.

Resolves BASELINE.json's prose exactly as SURVEY.md §8(d) fixes it (the reference
CLI cannot express these cells, `flapw.py:374-437`):

* cubic cell of side a, Omega = a^3, b = 2 pi / a;
* k = b (u - 1/2), u ~ U(0,1)^3 (C5: 64 points in the wedge 0 <= kz <= ky <= kx <= pi/a);
* G-set: integer triples n with |k + b n| <= K_max, K_max = (N_target 6 pi^2 / Omega)^(1/3)
  (the continuum rule of `flapw.py:402-403`), ordered by |K| then lexicographically
  (`flapw.py:415-417`);
* per type: positions U(0,1)^3 a, rotations = I, l_sph = l_nonsph = l_max, r_MT as
  given (C3/C5 do not state one: 2.2, C2's value); radial u, u', udot, udot' ~
  U(0.1, 1.0), ||udot|| = sqrt(U(0.01, 0.1)) (BASELINE draws ||udot||^2), energy 0;
* per type T blocks: X ~ CN(0,1); T_AA = (X + X^H)/(2 N_L) + 2 I, T_BB likewise with an
  independent X, T_AB = X'/N_L; all atoms of a type share the same T objects.

There is no dataset: the FLEUR NaCl/TiO2 inputs of the paper are not available, and
these seeded systems stand in for them.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .builder import TMatrixSet
from .flapw import RadialBoundaryData, SystemSpec
from .matrix import ComplexDense


@dataclass(frozen=True)
class ConfigDef:
    name: str
    cell: float
    n_target: int
    types: tuple      # ((n_atoms, r_mt), ...)
    l_max: int
    n_kpoints: int = 1
    seed: int = 0
    t_shift: float = 2.0
    l_nonsph: int | None = None  # None = l_max (BASELINE); else T is dense only in the leading
                                 # (l_nonsph+1)^2 block plus its diagonals
    bb_udot_scaled: bool = False  # T_BB -> U T_BB U (U = diag ||udot|| per row), as the physics
                                  # scales <udot|H|udot>


CONFIGS = {
    "C1": ConfigDef("C1", 8.0, 600, ((2, 2.0), (2, 2.2)), 6, seed=1001),
    "C2": ConfigDef("C2", 12.0, 3000, ((16, 2.2),), 8, seed=1002),
    "C3": ConfigDef("C3", 18.0, 8000, ((64, 2.2),), 8, seed=1003),
    "C4": ConfigDef("C4", 22.0, 13000, ((36, 2.0), (36, 2.2), (36, 2.4)), 10, seed=1004),
    "C5": ConfigDef("C5", 14.0, 5000, ((32, 2.2),), 8, n_kpoints=64, seed=1005),
    # Not a BASELINE config: C2 with the paper's l_nonsph = 6 < l_sph = 8 (PAPER.md:649-652,
    # :759-813), T zeroed outside the dense block except its diagonals as the reference's
    # synth_T does (`flapw.py:440-446` _fig1_zero_out): exercises the T-structure split.
    "C2NS": ConfigDef("C2NS", 12.0, 3000, ((16, 2.2),), 8, seed=1006, l_nonsph=6),
    # Not a BASELINE config: C2 with indefinite T (SURVEY §8d's test variant, diagonal -2) and
    # T_BB scaled by ||udot||: no T_AA is HPD; exercises the shifted joint H form.
    "C2IND": ConfigDef("C2IND", 12.0, 3000, ((16, 2.2),), 8, seed=1007, t_shift=-2.0,
                       bb_udot_scaled=True),
}


def _zero_outside(a: np.ndarray, d: int) -> np.ndarray:
    """Keep the leading d x d block and the diagonal (reference `_fig1_zero_out`)."""
    out = np.diag(np.diag(a)).astype(np.complex128)
    out[:d, :d] = a[:d, :d]
    return out


def g_set(k: np.ndarray, cell: float, n_target: int) -> np.ndarray:
    """K = k + G vectors inside the cutoff sphere, sorted by |K| then (n0, n1, n2)."""
    omega = cell**3
    b = 2.0 * np.pi / cell
    k_max = (n_target * 6.0 * np.pi**2 / omega) ** (1.0 / 3.0)
    n_max = int(np.ceil((k_max + np.linalg.norm(k)) / b)) + 1
    grid = np.arange(-n_max, n_max + 1)
    trip = np.stack(np.meshgrid(grid, grid, grid, indexing="ij"), axis=-1).reshape(-1, 3)
    kv = k[None, :] + b * trip
    norms = np.linalg.norm(kv, axis=1)
    keep = norms <= k_max
    kv, trip, norms = kv[keep], trip[keep], norms[keep]
    order = np.lexsort((trip[:, 2], trip[:, 1], trip[:, 0], norms))
    return kv[order]


def _kpoints(rng, cfg: ConfigDef) -> np.ndarray:
    b = 2.0 * np.pi / cfg.cell
    if cfg.n_kpoints == 1:
        return (b * (rng.uniform(0.0, 1.0, 3) - 0.5))[None, :]
    pts = []
    while len(pts) < cfg.n_kpoints:
        u = np.sort(rng.uniform(0.0, 0.5, 3))[::-1]  # kx >= ky >= kz >= 0, in units of b
        pts.append(b * u)
    return np.array(pts)


@dataclass
class Instance:
    """One seeded system: per-k-point specs sharing atoms/radial data, and the T set."""

    cfg: ConfigDef
    specs: list
    tmats: TMatrixSet
    min_abs_wronskian: float

    @property
    def spec(self) -> SystemSpec:
        return self.specs[0]


def make_instance(name: str, seed: int | None = None, n_kpoints: int | None = None,
                  hpd_shift: float | None = None) -> Instance:
    cfg = CONFIGS[name]
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    kpts = _kpoints(rng, cfg)
    if n_kpoints is not None:
        kpts = kpts[:n_kpoints]
    n_l = (cfg.l_max + 1) ** 2
    shift = cfg.t_shift if hpd_shift is None else hpd_shift
    l_ns = cfg.l_max if cfg.l_nonsph is None else cfg.l_nonsph
    positions, rmt, radial, t_aa, t_ab, t_bb = [], [], [], [], [], []
    wmin = np.inf
    for n_atoms, r_mt in cfg.types:
        pos = rng.uniform(0.0, 1.0, (n_atoms, 3)) * cfg.cell
        vals = rng.uniform(0.1, 1.0, (4, cfg.l_max + 1))
        udot_norm = np.sqrt(rng.uniform(0.01, 0.1, cfg.l_max + 1))
        rad = RadialBoundaryData(u=vals[0], u_prime=vals[1], udot=vals[2], udot_prime=vals[3],
                                 energy=np.zeros(cfg.l_max + 1), udot_norm=udot_norm)
        wmin = min(wmin, float(np.min(np.abs(rad.wronskian))))

        def cgauss():
            return rng.standard_normal((n_l, n_l)) + 1j * rng.standard_normal((n_l, n_l))

        x = cgauss()
        taa_a = (x + x.conj().T) / (2 * n_l) + shift * np.eye(n_l)
        x = cgauss()
        tbb_a = (x + x.conj().T) / (2 * n_l) + shift * np.eye(n_l)
        tab_a = cgauss() / n_l
        if l_ns < cfg.l_max:
            d = (l_ns + 1) ** 2
            taa_a, tbb_a, tab_a = (_zero_outside(t, d) for t in (taa_a, tbb_a, tab_a))
        if cfg.bb_udot_scaled:
            u_rows = np.repeat(udot_norm, 2 * np.arange(cfg.l_max + 1) + 1)
            tbb_a = u_rows[:, None] * tbb_a * u_rows[None, :]
        taa = ComplexDense.from_array(taa_a)
        tbb = ComplexDense.from_array(tbb_a)
        tab = ComplexDense.from_array(tab_a)
        for p in pos:
            positions.append(p)
            rmt.append(r_mt)
            radial.append(rad)
            t_aa.append(taa)
            t_ab.append(tab)
            t_bb.append(tbb)
    n_at = len(positions)
    l_arr = np.full(n_at, cfg.l_max, dtype=np.int64)
    specs = []
    for k in kpts:
        specs.append(SystemSpec(
            positions=np.array(positions), rotations=np.tile(np.eye(3), (n_at, 1, 1)),
            mt_radius=np.array(rmt), l_sph=l_arr, l_nonsph=np.full(n_at, l_ns, dtype=np.int64), k_point=k,
            k_vectors=g_set(k, cfg.cell, cfg.n_target), omega=cfg.cell**3, radial=radial))
    tm = TMatrixSet(t_aa=t_aa, t_ab=t_ab, t_bb=t_bb, l_sph=[cfg.l_max] * n_at,
                    l_nonsph=[l_ns] * n_at)
    return Instance(cfg, specs, tm, wmin)


def nominal_flops(spec: SystemSpec, hpd_mask=None) -> int:
    """Reference ledger total (`builder.py:336-370`) for one k-point of this spec."""
    from .builder import predict_flops

    heights = [int((l + 1) ** 2) for l in spec.l_sph]
    mask = [True] * len(heights) if hpd_mask is None else hpd_mask
    return predict_flops(len(heights), heights, spec.n_basis, mask).total


def kpoint_variant(inst: Instance, index: int) -> SystemSpec:
    """The instance's system at another seeded k-point (index 0 = the instance's own).

    Used for k-point weak scaling: rank r of a multi-GPU run handles its own k-point of
    the same crystal (atoms, radial data and T blocks shared)."""
    if index < len(inst.specs):
        return inst.specs[index]
    cfg = inst.cfg
    rng = np.random.default_rng(cfg.seed * 7919 + index)
    b = 2.0 * np.pi / cfg.cell
    k = b * (np.sort(rng.uniform(0.0, 0.5, 3))[::-1] if cfg.n_kpoints > 1
             else rng.uniform(0.0, 1.0, 3) - 0.5)
    base = inst.specs[0]
    return SystemSpec(positions=base.positions, rotations=base.rotations,
                      mt_radius=base.mt_radius, l_sph=base.l_sph, l_nonsph=base.l_nonsph,
                      k_point=k, k_vectors=g_set(k, cfg.cell, cfg.n_target), omega=base.omega,
                      radial=base.radial)
