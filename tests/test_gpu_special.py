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
