"""H through the joint factor of each T set's 2m x 2m matrix [[T_AA, T_AB], [T_AB^H, T_BB]]
(hsdla_build_args.h_reference_form = 0, the default): where that matrix is HPD, L L^H = it and
the atom's whole H contribution is W^H W with W = L^H [A_a; B_a] — one stacked rank-2R update
instead of the reference's ZHER2K + ZHERK (builder.py:212-315).  Checked against the oracle
(pinned to the reference's goldens) and against the reference forms Z / Y / X on the same
device, for joint-HPD sets, sets where only T_AA is HPD (fallback to Y), non-HPD T_AA
(fallback to X), T smaller than its block, and the forced general path."""
import numpy as np
import pytest

from conftest import rand_complex, rel_fro
from oracle import build as ob

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def pkg(cuda):
    import paper_1602_06589_b200 as p

    p._native.load()
    return p


def _hermitian(rng, m, shift):
    x = rand_complex(rng, m, m)
    return (x + x.conj().T) / (2 * m) + shift * np.eye(m)


def _case(pkg, seed, heights, n_g, t_sizes, aa_shifts, bb_shifts):
    rng = np.random.default_rng(seed)
    lay = pkg.AtomBlockLayout(tuple(heights))
    r = lay.total_rows
    a = pkg.ComplexDense.zeros(r, n_g, capacity_rows=lay.capacity_rows)
    b = pkg.ComplexDense.zeros(r, n_g, capacity_rows=lay.capacity_rows)
    a.array[:] = rand_complex(rng, r, n_g)
    b.array[:] = rand_complex(rng, r, n_g)
    u = rng.uniform(0.2, 1.5, r)
    co = pkg.StackedCoefficients(a, b, lay, u)
    taa = [_hermitian(rng, m, s) for m, s in zip(t_sizes, aa_shifts)]
    tbb = [_hermitian(rng, m, s) for m, s in zip(t_sizes, bb_shifts)]
    tab = [rand_complex(rng, m, m) / m for m in t_sizes]
    # poison the strict upper triangles (read from the lower only) and diagonal imaginaries
    for t in taa + tbb:
        t[np.triu_indices(len(t), 1)] = np.nan
        t[np.diag_indices(len(t))] += 3.0j
    cd = pkg.ComplexDense.from_array
    tm = pkg.TMatrixSet([cd(t) for t in taa], [cd(t) for t in tab], [cd(t) for t in tbb],
                        [0] * len(heights), [0] * len(heights))
    herm = [np.tril(t, -1) + np.tril(t, -1).conj().T + np.diag(t.diagonal().real) for t in taa]
    hbb = [np.tril(t, -1) + np.tril(t, -1).conj().T + np.diag(t.diagonal().real) for t in tbb]
    return co, tm, (a.array.copy(), b.array.copy(), u.copy(), herm, tab, hbb)


def _build(pkg, co, tm, force=False, reference_form=False, shift=False):
    import torch

    from paper_1602_06589_b200 import device
    from paper_1602_06589_b200.pipeline import build_device, pack_tmats, padded_ld

    lay, n = co.layout, co.n_basis
    r = lay.total_rows
    ld = padded_ld(r)
    a_d = device.upload_window(co.A_star.array, ld)
    b_d = device.upload_window(co.B_star.array, ld)
    udot = torch.zeros(ld, dtype=torch.float64, device="cuda")
    udot[:r] = torch.from_numpy(np.ascontiguousarray(co.udot_norms)).cuda()
    h_d, s_d = device.empty_matrix(n, n, n), device.empty_matrix(n, n, n)
    res, _ = build_device(n_basis=n, heights=lay.block_heights, row_offset=lay.offsets[:-1],
                          tpack=pack_tmats(tm), A=a_d, B=b_d, Bs=None, udot=udot, ld=ld,
                          force_general_path=force, H=h_d, S=s_d, ldh=n,
                          h_reference_form=reference_form,
                          udot_rows=np.asarray(co.udot_norms) if shift else None)
    torch.cuda.synchronize()
    return h_d.cpu().numpy().T.copy(), s_d.cpu().numpy().T.copy(), res


def _check(pkg, co, tm, ref, want_joint, want_hpd, force=False):
    a, b, u, taa, tab, tbb = ref
    heights = list(co.layout.block_heights)
    h_o, s_o, _, mask_o = ob.build_all(a, b, u, heights, taa, tab, tbb, force_general_path=force)
    h, s, res = _build(pkg, co, tm, force=force)
    h_r, s_r, res_r = _build(pkg, co, tm, force=force, reference_form=True)
    assert res["joint_t"] == want_joint
    assert res_r["joint_t"] == [False] * len(want_joint)
    assert res["hpd_mask"] == res_r["hpd_mask"] == want_hpd == list(mask_o)
    assert rel_fro(h, h_o) <= TOL and rel_fro(s, s_o) <= TOL
    assert rel_fro(h, h_r) <= 1e-13
    np.testing.assert_array_equal(s, s_r)  # S does not depend on the H form
    np.testing.assert_array_equal(h, h.conj().T)
    return h, h_r


def test_joint_form_all_hpd(pkg):
    heights = (9, 9, 9, 9)
    co, tm, ref = _case(pkg, 1, heights, 130, [9] * 4, [2.0] * 4, [2.0] * 4)
    h, h_r = _check(pkg, co, tm, ref, [True] * 4, [True] * 4)
    assert not np.array_equal(h, h_r)  # the two forms really are different evaluations


def test_joint_form_mixed_fallbacks(pkg):
    """Set 0 joint-HPD; set 1: T_AA HPD but T_BB = -2 I-ish (joint not HPD -> Y path);
    set 2: T_AA not HPD (X path); set 3: joint-HPD with T smaller than its block."""
    heights = (16, 16, 9, 25)
    co, tm, ref = _case(pkg, 2, heights, 97, [16, 16, 9, 16], [2.0, 2.0, -2.0, 2.0],
                        [2.0, -2.0, 2.0, 1.5])
    _check(pkg, co, tm, ref, [True, False, False, True], [True, True, False, True])


def test_joint_form_forced_general_path(pkg):
    heights = (9, 16)
    co, tm, ref = _case(pkg, 3, heights, 70, [9, 16], [2.0, 2.0], [2.0, 2.0])
    _check(pkg, co, tm, ref, [False, False], [False, False], force=True)


def test_joint_form_shared_type_pipeline_reuse(pkg):
    """BASELINE-style shared type (C1): every atom joint; a k-point batch reuses the cached
    joint factor (no second T preparation) and equals single builds bitwise."""
    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.pipeline import build_hs, build_hs_many

    inst = configs.make_instance("C1")
    h1, s1, r1 = build_hs(inst.spec, inst.tmats)
    assert all(r1["joint_t"])
    out = {}
    rr = build_hs_many([inst.spec] * 3, inst.tmats,
                       on_result=lambda i, h, s, r: out.__setitem__(i, (h.array.copy(), s.array.copy())))
    assert all(all(r["joint_t"]) for r in rr)
    for i in range(3):
        np.testing.assert_array_equal(out[i][0], h1.array)
        np.testing.assert_array_equal(out[i][1], s1.array)


def _structured(rng, m, d, shift):
    """Dense d x d Hermitian block + real diagonal tail (assemble_T's shape, flapw.py:306-363)."""
    t = np.zeros((m, m), dtype=np.complex128)
    t[:d, :d] = _hermitian(rng, d, 0.0)
    t[np.diag_indices(m)] += shift + rng.uniform(-0.2, 0.2, m)
    return t


def _split_case(pkg, seed, heights, d_sizes, n_g, tail_bb=1.5, break_structure=False):
    rng = np.random.default_rng(seed)
    lay = pkg.AtomBlockLayout(tuple(heights))
    r = lay.total_rows
    a = pkg.ComplexDense.zeros(r, n_g, capacity_rows=lay.capacity_rows)
    b = pkg.ComplexDense.zeros(r, n_g, capacity_rows=lay.capacity_rows)
    a.array[:] = rand_complex(rng, r, n_g)
    b.array[:] = rand_complex(rng, r, n_g)
    u = rng.uniform(0.2, 1.5, r)
    co = pkg.StackedCoefficients(a, b, lay, u)
    taa, tab, tbb = [], [], []
    for m, d in zip(heights, d_sizes):
        taa.append(_structured(rng, m, d, 2.0))
        tbb.append(_structured(rng, m, d, tail_bb))
        x = np.zeros((m, m), dtype=np.complex128)
        x[:d, :d] = rand_complex(rng, d, d) / m
        x[np.diag_indices(m)] += 1.0  # assemble_T's unit AB diagonal
        tab.append(x)
    if break_structure:
        tab[0][heights[0] - 1, 0] = 1e-3
    cd = pkg.ComplexDense.from_array
    l_sph = [int(round(np.sqrt(m))) - 1 for m in heights]
    l_ns = [int(round(np.sqrt(d))) - 1 for d in d_sizes]
    tm = pkg.TMatrixSet([cd(t) for t in taa], [cd(t) for t in tab], [cd(t) for t in tbb],
                        l_sph, l_ns)
    return co, tm, (a.array.copy(), b.array.copy(), u.copy(), taa, tab, tbb)


def test_joint_structure_split(pkg):
    """l_sph = 8, l_nonsph = 6 (the paper's case) and l_sph = 4, l_nonsph = 2: T dense in its
    leading (l_nonsph+1)^2 block plus diagonals -> 2d x 2d joint factor, 2x2 per tail row, T
    applications with K = d and an elementwise tail; equal to the dense forms and the oracle."""
    heights, dense = (81, 81, 25), (49, 49, 9)
    co, tm, ref = _split_case(pkg, 21, heights, dense, 173)
    h, h_r = _check(pkg, co, tm, ref, [True] * 3, [True] * 3)
    from paper_1602_06589_b200.pipeline import build_device  # noqa: F401
    _, _, res = _build(pkg, co, tm)
    assert res["joint_split"] == [True] * 3


def test_joint_structure_split_fallbacks(pkg):
    """An off-structure entry disables the split for that set (dense joint factor instead);
    a tail 2x2 block that is not HPD (T_BB tail below |T_AB|^2 / T_AA) sends the set to the
    reference forms."""
    heights, dense = (25, 25), (9, 9)
    co, tm, ref = _split_case(pkg, 22, heights, dense, 90, break_structure=True)
    _, _, res = _build(pkg, co, tm)
    assert res["joint_t"] == [True, True] and res["joint_split"] == [False, True]
    _check(pkg, co, tm, ref, [True, True], [True, True])
    co, tm, ref = _split_case(pkg, 23, heights, dense, 90, tail_bb=0.1)
    _, _, res = _build(pkg, co, tm)
    assert res["joint_t"] == [False, False]
    _check(pkg, co, tm, ref, [False, False], [True, True])


def test_joint_form_large_blocks(pkg):
    """l_sph = 12 and 11 blocks (m = 169, 144): the joint factor's 2m exceeds the packed
    shared-memory Cholesky (column kernel in global memory) and the T applications run on
    64-row tiles; mixed with a small set (mixed packed / column choice per launch)."""
    heights = (169, 144, 16)
    co, tm, ref = _case(pkg, 4, heights, 150, list(heights), [2.0, 2.0, 2.0], [2.0, 2.0, 2.0])
    _check(pkg, co, tm, ref, [True, True, True], [True, True, True])


def test_assemble_t_output_through_the_build(pkg):
    """T from the GPU assemble_T (Gaunt sums, reference golden integrals): with energies shifted
    up the joint matrix is HPD and the build takes the structure split; as generated (energies in
    [-1, 1]) it takes the reference forms.  Both against the oracle."""
    from types import SimpleNamespace

    from conftest import golden

    d = golden("assemble_t.npz")
    n = len(d["l_sph"])
    ris = [pkg.RadialIntegrals(d[f"c_uu{a}"], d[f"c_dd{a}"], d[f"c_ud{a}"], d[f"c_du{a}"])
           for a in range(n)]
    heights = tuple(int((l + 1) ** 2) for l in d["l_sph"])
    for shift, want_split in ((12.0, True), (0.0, None)):
        radial = [SimpleNamespace(energy=d[f"energy{a}"] + shift, udot_norm=d[f"udot_norm{a}"])
                  for a in range(n)]
        spec = SimpleNamespace(n_atoms=n, l_sph=d["l_sph"], l_nonsph=d["l_nonsph"], radial=radial)
        tm = pkg.assemble_T(spec, ris)
        rng = np.random.default_rng(5)
        lay = pkg.AtomBlockLayout(heights)
        r = lay.total_rows
        a = pkg.ComplexDense.zeros(r, 120, capacity_rows=lay.capacity_rows)
        b = pkg.ComplexDense.zeros(r, 120, capacity_rows=lay.capacity_rows)
        a.array[:] = rand_complex(rng, r, 120)
        b.array[:] = rand_complex(rng, r, 120)
        u = rng.uniform(0.2, 1.5, r)
        co = pkg.StackedCoefficients(a, b, lay, u)
        ref = (a.array.copy(), b.array.copy(), u.copy(), [t.array for t in tm.t_aa],
               [t.array for t in tm.t_ab], [t.array for t in tm.t_bb])
        h, s, res = _build(pkg, co, tm)
        h_o, s_o, _, mask_o = ob.build_all(*ref[:3], list(heights), *ref[3:])
        assert rel_fro(h, h_o) <= TOL and rel_fro(s, s_o) <= TOL
        assert res["hpd_mask"] == list(mask_o)
        if want_split:
            assert all(res["joint_t"])
            # l_nonsph < l_sph sets split; l_nonsph == l_sph (atom 1) has no tail
            assert res["joint_split"] == [bool(ln < ls) for ls, ln in zip(d["l_sph"], d["l_nonsph"])]



def _uniform_udot_case(pkg, seed, heights, n_g, aa_shifts, bb_shifts, u_range=(0.8, 1.2)):
    """_case with one ||udot|| row pattern per block height (atoms of a T set share it)."""
    co, tm, ref = _case(pkg, seed, heights, n_g, list(heights), aa_shifts, bb_shifts)
    rng = np.random.default_rng(seed + 100)
    pattern = {h: rng.uniform(*u_range, h) for h in set(heights)}
    u = np.concatenate([pattern[h] for h in heights])
    co.udot_norms[:] = u
    return co, tm, (ref[0], ref[1], u.copy()) + ref[3:]


def test_shifted_joint_form_indefinite_t(pkg):
    """T_AA / T_BB not HPD: the joint form with a common shift, H = sum W^H W - sigma S, against
    the oracle and the reference forms; every set joint, sigma > 0 (||udot|| ~ 1, so the shift
    is of the size of T and passes the amplification guard)."""
    heights = (16, 16, 9)
    co, tm, ref = _uniform_udot_case(pkg, 31, heights, 110, [-2.0, 2.0, -1.0], [2.0, -2.0, -0.5])
    a, b, u, taa, tab, tbb = ref
    h_o, s_o, _, mask_o = ob.build_all(a, b, u, list(heights), taa, tab, tbb)
    h, s, res = _build(pkg, co, tm, shift=True)
    h_r, _, res_r = _build(pkg, co, tm, reference_form=True)
    assert res["joint_t"] == [True] * 3 and res["joint_shift"] > 0
    assert res_r["joint_shift"] == 0 and res["hpd_mask"] == list(mask_o) == [False, True, False]
    assert rel_fro(h, h_o) <= TOL and rel_fro(s, s_o) <= TOL
    assert rel_fro(h, h_r) <= 1e-13
    np.testing.assert_array_equal(h, h.conj().T)


def test_shifted_joint_form_needs_uniform_udot(pkg):
    """Atoms of one T set with different ||udot|| rows (or T smaller than the block) cannot
    share a shift: non-HPD sets then take the reference forms, HPD sets stay joint unshifted."""
    heights = (16, 16)
    co, tm, ref = _uniform_udot_case(pkg, 32, heights, 90, [-2.0, 2.0], [2.0, 2.0])
    co.udot_norms[16] *= 1.5  # atom 1 (own T set) is fine; make atom 0's set share T with it
    tm = pkg.TMatrixSet([tm.t_aa[0]] * 2, [tm.t_ab[0]] * 2, [tm.t_bb[0]] * 2, [0, 0], [0, 0])
    a, b, _, taa, tab, tbb = ref
    u = np.asarray(co.udot_norms).copy()
    h_o, s_o, _, _ = ob.build_all(a, b, u, list(heights), [taa[0]] * 2, [tab[0]] * 2, [tbb[0]] * 2)
    h, s, res = _build(pkg, co, tm, shift=True)
    assert res["joint_t"] == [False] and res["joint_shift"] == 0
    assert rel_fro(h, h_o) <= TOL and rel_fro(s, s_o) <= TOL


def test_shifted_joint_form_guard_and_drop_in(pkg):
    """Badly scaled T (shift -2 on T_BB against ||udot||^2 ~ 0.05, BASELINE C1 with the test
    variant's diagonal -2): the needed shift would amplify rounding ~100x, so the guard keeps the
    reference forms — through the device pipeline and the drop-in build_all, both vs the oracle."""
    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.pipeline import build_hs

    inst = configs.make_instance("C1", hpd_shift=-2.0)
    h, s, res = build_hs(inst.spec, inst.tmats)
    assert not any(res["joint_t"]) and res["joint_shift"] == 0 and not any(res["hpd_mask"])
    co = pkg.compute_AB(inst.spec)
    h2, s2, rep = pkg.build_all(co, inst.tmats, pkg.BuildConfig())
    from oracle import flapw as of
    a, b, norms, offs = of.compute_ab(inst.spec)
    tm = inst.tmats
    h_o, s_o, _, mask = ob.build_all(a, b, norms, list(np.diff(offs)), [t.array for t in tm.t_aa],
                                     [t.array for t in tm.t_ab], [t.array for t in tm.t_bb])
    for hh, ss in ((h, s), (h2, s2)):
        assert rel_fro(hh.array, h_o) <= TOL and rel_fro(ss.array, s_o) <= TOL
    assert rep.hpd_mask == list(mask)


def test_shifted_joint_form_guard_small_udot(pkg):
    """The same indefinite T with ||udot|| ~ 0.2: the shift needed by the B blocks would be
    ~25x T's scale; rejected, the reference forms give H (vs the oracle)."""
    heights = (16, 9)
    co, tm, ref = _uniform_udot_case(pkg, 33, heights, 80, [2.0, 2.0], [-2.0, -1.0],
                                     u_range=(0.15, 0.25))
    a, b, u, taa, tab, tbb = ref
    h_o, s_o, _, _ = ob.build_all(a, b, u, list(heights), taa, tab, tbb)
    h, s, res = _build(pkg, co, tm, shift=True)
    assert res["joint_t"] == [False, False] and res["joint_shift"] == 0
    assert rel_fro(h, h_o) <= TOL and rel_fro(s, s_o) <= TOL
