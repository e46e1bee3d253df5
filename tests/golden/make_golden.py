"""Generate the golden fixtures by running the REAL reference package (build container only).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden.py

Imports `hsdla` from /root/reference/pkg/src (read-only; not available on the GPU box)
and writes small .npz fixtures next to this script:

* special.npz   — spherical_bessel_all / spherical_harmonics_all values (special.py:104-179)
* ab_small.npz  — compute_AB on a small spec with random rotations, mixed l_sph and a
                  K = 0 vector, full A*/B* (flapw.py:201-233)
* ab_high.npz   — compute_AB at l_sph 12..14 (the supported maximum), x = |K| r up to ~21
* reduced.npz   — reduced_overlap_inputs + reduced_S_AA on the small spec (full) and on
                  C1 (projections, diagonal, first column)
* ab_c1.npz     — compute_AB on BASELINE C1: sampled columns + projections A* V
* build_small.npz — build_all (optimized backend) on small mixed-HPD / varying-height
                  instances: inputs and full H, S, ledger, hpd mask (builder.py:403-474)
* build_c1.npz  — compute_AB + build_all on C1: H V, S V projections, diagonals,
                  Frobenius norms, ledger and mask

The fixtures pin both the oracle (tests/test_oracle_golden.py) and the GPU path
(tests/test_gpu_parity.py).  Re-run after changing configs.py (C1 inputs come from it).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import hsdla  # noqa: E402  (the reference)

from paper_1602_06589_b200 import configs  # noqa: E402


def ref_spec(spec):
    return hsdla.SystemSpec.from_json_dict(spec.to_json_dict())


def ref_tmats(tm):
    cd = hsdla.ComplexDense.from_array
    return hsdla.TMatrixSet(t_aa=[cd(t.array) for t in tm.t_aa], t_ab=[cd(t.array) for t in tm.t_ab],
                            t_bb=[cd(t.array) for t in tm.t_bb], l_sph=list(tm.l_sph),
                            l_nonsph=list(tm.l_nonsph))


def special():
    xs = np.array([0.0, 1e-3, 0.3, 0.49, 0.5, 1.0, 2.5, 5.0, 7.9, 8.0, 9.0, 10.5, 11.0, 15.0, 20.0])
    out = {"x": xs}
    for lm in (0, 1, 6, 8, 10, 12):
        js, jps = [], []
        for x in xs:
            j, jp = hsdla.spherical_bessel_all(lm, float(x))
            js.append(j)
            jps.append(jp)
        out[f"j_{lm}"] = np.array(js)
        out[f"jp_{lm}"] = np.array(jps)
    rng = np.random.default_rng(5)
    d = rng.standard_normal((50, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    d[0] = (0.0, 0.0, 1.0)
    d[1] = (0.0, 0.0, -1.0)
    d[2] = (1.0, 0.0, 0.0)
    out["dirs"] = d
    out["ylm_10"] = hsdla.spherical_harmonics_all(10, d)
    np.savez_compressed(os.path.join(HERE, "special.npz"), **out)


def small_spec(seed=3):
    rng = np.random.default_rng(seed)
    n_atoms = 4
    l_sph = np.array([0, 3, 6, 10])
    pos = rng.uniform(0, 1, (n_atoms, 3)) * 5.0
    rots = []
    for _ in range(n_atoms):
        q, r = np.linalg.qr(rng.standard_normal((3, 3)))
        q *= np.sign(np.diag(r))
        rots.append(q)
    rots[1] = -rots[1]  # an improper rotation (|det| = 1 allowed)
    kv = rng.standard_normal((40, 3)) * 2.0
    kv[0] = 0.0
    kv[1] = (0.0, 0.0, 0.1)
    kv[2] = (0.0, 0.0, -3.0)
    kv[3] = (1e-3, 0.0, 0.0)
    radial = []
    for a in range(n_atoms):
        n = l_sph[a] + 1
        radial.append(hsdla.RadialBoundaryData(
            u=rng.uniform(0.1, 1, n), u_prime=rng.uniform(0.1, 1, n), udot=rng.uniform(0.1, 1, n),
            udot_prime=rng.uniform(0.1, 1, n), energy=np.zeros(n),
            udot_norm=np.sqrt(rng.uniform(0.01, 0.1, n))))
    return hsdla.SystemSpec(positions=pos, rotations=np.array(rots),
                            mt_radius=np.array([2.0, 1.5, 2.4, 2.2]), l_sph=l_sph,
                            l_nonsph=l_sph, k_point=np.zeros(3), k_vectors=kv, omega=125.0,
                            radial=radial)


def spec_arrays(spec, prefix="spec_"):
    d = {f"{prefix}positions": spec.positions, f"{prefix}rotations": spec.rotations,
         f"{prefix}mt_radius": spec.mt_radius, f"{prefix}l_sph": spec.l_sph,
         f"{prefix}k_vectors": spec.k_vectors, f"{prefix}omega": np.array(spec.omega)}
    for f in ("u", "u_prime", "udot", "udot_prime", "udot_norm"):
        d[f"{prefix}rad_{f}"] = np.array([np.pad(getattr(r, f), (0, 16 - len(getattr(r, f))))
                                          for r in spec.radial])
    return d


def ab_small():
    spec = small_spec()
    c = hsdla.compute_AB(spec)
    out = spec_arrays(spec)
    out.update(A=c.A_star.array, B=c.B_star.array, udot_norms=c.udot_norms)
    np.savez_compressed(os.path.join(HERE, "ab_small.npz"), **out)


def high_spec():
    """Spec at the largest supported l (HSDLA_MAX_LSPH = 14) with |K| r_MT up to ~21, so all
    three Bessel regimes (series, Miller, upward) occur at l = 12..14."""
    rng = np.random.default_rng(9)
    l_sph = np.array([12, 14, 13])
    n_atoms = len(l_sph)
    pos = rng.uniform(0, 1, (n_atoms, 3)) * 6.0
    rots = np.array([np.eye(3), np.linalg.qr(rng.standard_normal((3, 3)))[0], np.eye(3)])
    kv = rng.standard_normal((60, 3))
    kv *= (rng.uniform(0.0, 8.5, 60) / np.linalg.norm(kv, axis=1))[:, None]
    kv[0] = 0.0
    kv[1] = (0.0, 0.0, 0.05)
    radial = []
    for a in range(n_atoms):
        n = l_sph[a] + 1
        radial.append(hsdla.RadialBoundaryData(
            u=rng.uniform(0.1, 1, n), u_prime=rng.uniform(0.1, 1, n), udot=rng.uniform(0.1, 1, n),
            udot_prime=rng.uniform(0.1, 1, n), energy=np.zeros(n),
            udot_norm=np.sqrt(rng.uniform(0.01, 0.1, n))))
    spec = hsdla.SystemSpec(positions=pos, rotations=rots, mt_radius=np.array([2.5, 2.2, 1.8]),
                            l_sph=l_sph, l_nonsph=l_sph, k_point=np.zeros(3), k_vectors=kv,
                            omega=216.0, radial=radial)
    return spec


def ab_high():
    """compute_AB on high_spec()."""
    spec = high_spec()
    c = hsdla.compute_AB(spec)
    out = spec_arrays(spec)
    out.update(A=c.A_star.array, B=c.B_star.array, udot_norms=c.udot_norms)
    np.savez_compressed(os.path.join(HERE, "ab_high.npz"), **out)


def reduced():
    """reduced_overlap_inputs + reduced_S_AA (flapw.py:236-250, oracle.py:159-216): the small
    mixed-l spec in full, C1 through projections."""
    out = {}
    spec = small_spec()
    inp = hsdla.reduced_overlap_inputs(spec)
    out.update(spec_arrays(spec))
    for a, (f, w) in enumerate(zip(inp.f, inp.wronskians)):
        out[f"small_f_{a}"], out[f"small_w_{a}"] = f, w
    out["small_S"] = hsdla.reduced_S_AA(inp).array
    c1spec = ref_spec(configs.make_instance("C1").spec)
    inp = hsdla.reduced_overlap_inputs(c1spec)
    s = hsdla.reduced_S_AA(inp).array
    v = projections(s.shape[0], seed=78)
    out.update(c1_f_0=inp.f[0], c1_V=v, c1_SV=s @ v, c1_diag=np.diag(s).copy(),
               c1_col0=s[:, 0].copy(), c1_fro=np.linalg.norm(s))
    np.savez_compressed(os.path.join(HERE, "reduced.npz"), **out)


def projections(n, k=6, seed=77):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))


def c1():
    inst = configs.make_instance("C1")
    spec = ref_spec(inst.spec)
    tm = ref_tmats(inst.tmats)
    coeffs = hsdla.compute_AB(spec)
    a, b = coeffs.A_star.array.copy(), coeffs.B_star.array.copy()
    n = a.shape[1]
    cols = np.arange(0, n, 7)
    v = projections(n)
    np.savez_compressed(os.path.join(HERE, "ab_c1.npz"), cols=cols, A_cols=a[:, cols],
                        B_cols=b[:, cols], AV=a @ v, BV=b @ v, V=v, udot_norms=coeffs.udot_norms,
                        A_fro=np.linalg.norm(a), B_fro=np.linalg.norm(b))
    h, s, rep = hsdla.build_all(coeffs, tm, hsdla.BuildConfig(backend="optimized", thread_count=1))
    hh, ss = h.array, s.array
    np.savez_compressed(os.path.join(HERE, "build_c1.npz"), V=v, HV=hh @ v, SV=ss @ v,
                        H_diag=np.diag(hh).copy(), S_diag=np.diag(ss).copy(),
                        H_col0=hh[:, 0].copy(), S_col0=ss[:, 0].copy(),
                        H_fro=np.linalg.norm(hh), S_fro=np.linalg.norm(ss),
                        ledger=np.array([rep.ledger.as_dict()[k] for k in LEDGER_KEYS]),
                        hpd_mask=np.array(rep.hpd_mask))


LEDGER_KEYS = ("hermitian_rank_k", "hermitian_rank_2k", "general_product", "hermitian_product",
               "triangular_product", "cholesky", "row_scale")


def build_small():
    cases = []
    # (seed, heights, capacity, n_g, l_nonsph, hpd_fraction, force_general)
    specs = [(7, (4, 9, 9), 9, 16, [1, 2, 2], 0.0, False),
             (21, (4, 9), 9, 14, [1, 1], 0.5, False),
             (31, (9, 9), 9, 20, [2, 2], 1.0, False),
             (31, (9, 9), 9, 20, [2, 2], 1.0, True),
             (61, (4, 9, 16, 9), 16, 18, [1, 1, 2, 2], 0.5, False),
             (41, (1, 9, 4), 9, 12, [0, 2, 1], 0.0, False),
             (51, (9, 9, 9, 9), 9, 30, [1, 1, 1, 1], 0.5, False)]
    out = {}
    for ci, (seed, heights, cap, n_g, l_ns, frac, force) in enumerate(specs):
        lay = hsdla.AtomBlockLayout(heights, cap)
        coeffs = hsdla.synth_coefficients(seed, lay, n_g)
        tm = hsdla.synth_T(seed + 1, lay, l_ns, hpd_fraction=frac)
        pre = coeffs.copy()
        h, s, rep = hsdla.build_all(coeffs, tm, hsdla.BuildConfig(force_general_path=force))
        p = f"c{ci}_"
        out[p + "heights"] = np.array(heights)
        out[p + "cap"] = np.array(cap)
        out[p + "force"] = np.array(force)
        out[p + "A"] = pre.A_star.array
        out[p + "B"] = pre.B_star.array
        out[p + "udot"] = pre.udot_norms
        for fam in ("t_aa", "t_ab", "t_bb"):
            for a, t in enumerate(getattr(tm, fam)):
                out[f"{p}{fam}_{a}"] = t.array
        out[p + "H"] = h.array
        out[p + "S"] = s.array
        out[p + "ledger"] = np.array([rep.ledger.as_dict()[k] for k in LEDGER_KEYS])
        out[p + "hpd_mask"] = np.array(rep.hpd_mask)
        cases.append(ci)
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "build_small.npz"), **out)


def match():
    """match_factors (flapw.py:179-198): f_A and f_B of every atom of the small spec (all l up to
    10) and of ab_high's spec (l 12..14, every Bessel regime), from the reference itself."""
    out = {}
    for tag, spec in (("small", small_spec()), ("high", high_spec())):
        out.update({f"{tag}_{k}": v for k, v in spec_arrays(spec).items()})
        for a in range(spec.n_atoms):
            fa, fb = hsdla.flapw.match_factors(spec, a)
            out[f"{tag}_fa_{a}"] = fa
            out[f"{tag}_fb_{a}"] = fb
    np.savez_compressed(os.path.join(HERE, "match.npz"), **out)


if __name__ == "__main__":
    steps = {"special": special, "ab_small": ab_small, "ab_high": ab_high,
             "build_small": build_small, "c1": c1, "reduced": reduced, "match": match}
    for name in (sys.argv[1:] or list(steps)):  # e.g. `make_golden.py ab_high`
        steps[name]()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
