"""Per-type phase-factorised H and S against the stacked build,
which is itself pinned to the reference: shared-type systems (C1, C2), all-distinct atoms
(random rotations: one rank-1 phase Gram per atom), non-HPD T and the forced general path."""
import numpy as np
import pytest

from conftest import golden, rel_fro, spec_from_golden

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def pkg(cuda):
    import paper_1602_06589_b200 as p

    p._native.load()
    return p


def _check(pkg, spec, tmats, config=None):
    from paper_1602_06589_b200.factorized import build_hs_factorized
    from paper_1602_06589_b200.pipeline import build_hs

    config = config or pkg.BuildConfig()
    h, s, rep = build_hs_factorized(spec, tmats, config)
    h0, s0, res = build_hs(spec, tmats, config)
    assert rel_fro(h.array, h0.array) <= TOL, rel_fro(h.array, h0.array)
    assert rel_fro(s.array, s0.array) <= TOL, rel_fro(s.array, s0.array)
    np.testing.assert_array_equal(h.array, h.array.conj().T)
    assert rep.hpd_mask == res["hpd_mask"]
    return rep


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_factorized_matches_stacked_on_configs(pkg, name):
    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.factorized import atom_types

    inst = configs.make_instance(name)
    assert len(atom_types(inst.spec, inst.tmats)) < inst.spec.n_atoms  # shared types
    _check(pkg, inst.spec, inst.tmats)


def test_factorized_all_distinct_atoms_and_non_hpd(pkg):
    """Random rotations (ab_small spec): every atom is its own type; T_AA of atom 1 is not
    HPD; and the forced general path."""
    d = golden("ab_small.npz")
    spec = spec_from_golden(d)
    rng = np.random.default_rng(8)
    cd = pkg.ComplexDense.from_array
    t_aa, t_ab, t_bb = [], [], []
    for a, l in enumerate(spec.l_sph):
        m = (int(l) + 1) ** 2
        x = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
        t_aa.append(cd((x + x.conj().T) / (2 * m) + (-2.0 if a == 1 else 2.0) * np.eye(m)))
        y = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
        t_bb.append(cd((y + y.conj().T) / (2 * m) + np.eye(m)))
        t_ab.append(cd((rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / m))
    tm = pkg.TMatrixSet(t_aa, t_ab, t_bb, list(spec.l_sph), list(spec.l_sph))
    from paper_1602_06589_b200.factorized import atom_types

    assert len(atom_types(spec, tm)) == spec.n_atoms
    rep = _check(pkg, spec, tm)
    assert rep.hpd_mask[1] is False and rep.hpd_mask[0] is True
    _check(pkg, spec, tm, pkg.BuildConfig(force_general_path=True))
