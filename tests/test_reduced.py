"""Legendre-reduced A-side overlap (reference oracle.py:159-216, flapw.py:236-250) on the GPU.

Pinned to the reference's own reduced_overlap_inputs / reduced_S_AA outputs
(tests/golden/reduced.npz) and cross-checked against the stacked contraction A*^H A*.
"""
import numpy as np
import pytest

from conftest import golden, rel_fro, spec_from_golden

from paper_1602_06589_b200 import ContractViolationError
from paper_1602_06589_b200.reduced import (ReducedOverlapInputs, reduced_overlap_inputs,
                                           reduced_S_AA)

TOL = 1e-12


def test_inputs_validation():
    f = [np.ones((2, 3))]
    with pytest.raises(ContractViolationError):
        ReducedOverlapInputs(f, [np.array([1.0, 0.0])], np.zeros((1, 3)), np.ones((3, 3)), 1.0)
    with pytest.raises(ContractViolationError):
        ReducedOverlapInputs(f, [np.ones(2)], np.zeros((1, 3)), np.ones((3, 3)), 0.0)
    with pytest.raises(ContractViolationError):
        ReducedOverlapInputs(f, [np.ones(2)], np.zeros((2, 3)), np.ones((3, 3)), 1.0)


@pytest.mark.gpu
def test_match_factors_vs_reference(cuda):
    d = golden("reduced.npz")
    inp = reduced_overlap_inputs(spec_from_golden(d))
    for a in range(len(inp.f)):
        assert rel_fro(inp.f[a], d[f"small_f_{a}"]) <= 1e-13, a
        np.testing.assert_array_equal(inp.wronskians[a], d[f"small_w_{a}"])


@pytest.mark.gpu
def test_reduced_s_aa_small_vs_reference(cuda):
    d = golden("reduced.npz")
    spec = spec_from_golden(d)
    f = [d[f"small_f_{a}"] for a in range(spec.n_atoms)]
    w = [d[f"small_w_{a}"] for a in range(spec.n_atoms)]
    s = reduced_S_AA(ReducedOverlapInputs(f, w, spec.positions, spec.k_vectors, spec.omega)).array
    assert rel_fro(s, d["small_S"]) <= TOL
    np.testing.assert_array_equal(s, s.conj().T)   # exactly Hermitian by construction


@pytest.mark.gpu
def test_reduced_s_aa_c1_vs_reference_and_stacked(cuda):
    """C1 end to end on the GPU: reduced_overlap_inputs -> reduced_S_AA against the
    reference's projections, and against A*^H A* from compute_AB + the DMMA contraction."""
    import paper_1602_06589_b200 as p
    from paper_1602_06589_b200 import configs

    d = golden("reduced.npz")
    spec = configs.make_instance("C1").spec
    inp = reduced_overlap_inputs(spec)
    assert rel_fro(inp.f[0], d["c1_f_0"]) <= 1e-13
    s = reduced_S_AA(inp).array
    assert rel_fro(s @ d["c1_V"], d["c1_SV"]) <= TOL
    assert rel_fro(np.diag(s), d["c1_diag"]) <= TOL
    assert rel_fro(s[:, 0], d["c1_col0"]) <= TOL
    coeffs = p.compute_AB(spec)
    n = coeffs.n_basis
    acc = p.HermitianAccumulator(n)
    p.get_backend("b200").hermitian_rank_k_update(acc, coeffs.A_star, p.FlopLedger())
    stacked = acc.mirror_to_full().array
    assert rel_fro(s, stacked) <= TOL


@pytest.mark.gpu
def test_reduced_s_aa_high_l_matches_stacked(cuda):
    """l = 12..14 with rotated atoms: the addition theorem is rotation invariant, so the
    reduced sum must equal A*^H A* of the rotated-frame coefficients."""
    import paper_1602_06589_b200 as p

    spec = spec_from_golden(golden("ab_high.npz"))
    s = reduced_S_AA(reduced_overlap_inputs(spec)).array
    coeffs = p.compute_AB(spec)
    acc = p.HermitianAccumulator(coeffs.n_basis)
    p.get_backend("b200").hermitian_rank_k_update(acc, coeffs.A_star, p.FlopLedger())
    assert rel_fro(s, acc.mirror_to_full().array) <= 1e-11
