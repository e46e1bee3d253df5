"""The A/B generator's special functions and match factors as standalone GPU entry points
(reference special.py:104-186, flapw.py:179-198) against the reference's golden tables."""
import numpy as np
import pytest

from conftest import golden, rel_fro, spec_from_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg(cuda):
    import paper_1602_06589_b200 as p

    p._native.load()
    return p


def test_bessel_vs_reference_tables(pkg):
    """Every regime (x = 0, series, Miller, upward) at orders 0..12."""
    d = golden("special.npz")
    for lm in (0, 1, 6, 8, 10, 12):
        j, jp = pkg.spherical_bessel_all(lm, d["x"])
        np.testing.assert_allclose(j.T, d[f"j_{lm}"], rtol=1e-14, atol=1e-16)
        np.testing.assert_allclose(jp.T, d[f"jp_{lm}"], rtol=1e-14, atol=1e-16)
    j, jp = pkg.spherical_bessel_all(3, 0.0)  # scalar form and the exact x = 0 limits
    assert j.shape == (4,) and j[0] == 1.0 and not j[1:].any() and jp[1] == 1.0 / 3.0
    with pytest.raises(pkg.ContractViolationError):
        pkg.spherical_bessel_all(2, -1.0)
    with pytest.raises(pkg.ContractViolationError):
        pkg.spherical_bessel_all(15, 1.0)


def test_ylm_vs_reference_table(pkg):
    d = golden("special.npz")
    y = pkg.spherical_harmonics_all(10, d["dirs"])
    assert np.max(np.abs(y - d["ylm_10"])) <= 1e-14
    assert abs(pkg.spherical_harmonic(0, 0, [0.0, 0.0, 1.0]) - 0.28209479177387814) == 0.0
    with pytest.raises(pkg.ContractViolationError):
        pkg.spherical_harmonics_all(2, [[1.0, 1.0, 0.0]])


def test_match_factors_vs_reference(pkg):
    d = golden("reduced.npz")
    spec = spec_from_golden(d)
    for a in range(spec.n_atoms):
        fa, fb = pkg.match_factors(spec, a)
        assert rel_fro(fa, d[f"small_f_{a}"]) <= 1e-13
        assert fb.shape == fa.shape


@pytest.mark.parametrize("tag", ["small", "high"])
def test_match_factors_fa_fb_vs_reference(pkg, tag):
    """f_A and f_B on the device vs the reference's match_factors (match.npz), every atom,
    l up to 14 and all Bessel regimes, per l row (small Wronskians do not enter here)."""
    d = golden("match.npz")
    spec = spec_from_golden(d, prefix=f"{tag}_spec_")
    for a in range(spec.n_atoms):
        fa, fb = pkg.match_factors(spec, a)
        for f, ref in ((fa, d[f"{tag}_fa_{a}"]), (fb, d[f"{tag}_fb_{a}"])):
            assert f.shape == ref.shape
            for l in range(ref.shape[0]):
                assert rel_fro(f[l], ref[l]) <= 1e-13, (a, l)


def test_gpu_gaunt_and_assemble_t_vs_reference(cuda):
    """gaunt / gaunt_tensor / assemble_T on the GPU against the reference's
    own outputs (tests/golden/assemble_t.npz), plus assemble_T's validation errors."""
    from types import SimpleNamespace

    import paper_1602_06589_b200 as pkg

    d = golden("assemble_t.npz")
    assert np.max(np.abs(pkg.gaunt_tensor(3, 2) - d["g32"])) <= 1e-14
    assert np.max(np.abs(pkg.gaunt_tensor(2, 2) - d["g22"])) <= 1e-14
    for row, want, want2 in zip(d["gaunt_args"], d["gaunt_vals"], d["gaunt_vals_refine2"]):
        lp, mp, l, m, lpp, mpp = (int(x) for x in row)
        assert abs(pkg.gaunt((lp, mp), (l, m), (lpp, mpp)) - want) <= 1e-14
        assert abs(pkg.gaunt((lp, mp), (l, m), (lpp, mpp), refine=2) - want2) <= 1e-14
    n = len(d["l_sph"])
    radial = [SimpleNamespace(energy=d[f"energy{a}"], udot_norm=d[f"udot_norm{a}"]) for a in range(n)]
    spec = SimpleNamespace(n_atoms=n, l_sph=d["l_sph"], l_nonsph=d["l_nonsph"], radial=radial)
    ris = [pkg.RadialIntegrals(d[f"c_uu{a}"], d[f"c_dd{a}"], d[f"c_ud{a}"], d[f"c_du{a}"])
           for a in range(n)]
    tm = pkg.assemble_T(spec, ris)
    for a in range(n):
        for got, key in ((tm.t_aa[a], "t_aa"), (tm.t_ab[a], "t_ab"), (tm.t_bb[a], "t_bb")):
            want = d[f"{key}{a}"]
            assert np.max(np.abs(got.array - want)) <= 1e-13 * max(1.0, np.max(np.abs(want)))
    # the reference's generator gives the same integrals for the same seed
    ri0 = pkg.synth_radial_integrals(40, int(d["l_nonsph"][0]))
    np.testing.assert_allclose(ri0.c_uu, d["c_uu0"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(ri0.c_du, d["c_du0"], rtol=0, atol=1e-15)
    bad = pkg.RadialIntegrals(d["c_uu0"] + 0.1, d["c_dd0"], d["c_ud0"], d["c_du0"])
    with pytest.raises(pkg.ContractViolationError):
        pkg.assemble_T(spec, [bad] + ris[1:])
    with pytest.raises(pkg.ContractViolationError):
        pkg.assemble_T(spec, ris[:2])
