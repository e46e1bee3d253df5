"""GPU parity: the sm_100a path (through libhsdla_b200.so's C ABI) against the oracle
and the golden vectors made by the real reference.  Tolerances are relative Frobenius
errors; the north_star bar is <= 1e-12 for H and S on every config."""
import numpy as np
import pytest

from conftest import (LEDGER_KEYS, build_case, golden, hermitian_from_lower, rand_complex,
                      rel_fro, spec_from_golden)
from oracle import build as ob
from oracle import flapw as of

pytestmark = pytest.mark.gpu

TOL = 1e-12  # north_star parity bar for H and S (relative Frobenius)


@pytest.fixture(scope="module")
def pkg(cuda):
    import paper_1602_06589_b200 as p

    p._native.load()
    return p


# ---------------------------------------------------------------- operators

@pytest.mark.parametrize("k,n", [(1, 2), (98, 64), (6, 5), (300, 257), (17, 129), (1296, 200)])
def test_herk_lower_vs_numpy(pkg, k, n):
    rng = np.random.default_rng(k * 1000 + n)
    a = rand_complex(rng, k, n)
    c0 = np.tril(rand_complex(rng, n, n))
    acc = pkg.HermitianAccumulator(n)
    acc.matrix.array[:] = c0
    iu = np.triu_indices(n, 1)
    acc.matrix.array[iu] = np.nan  # strict upper poison must survive untouched
    pkg.get_backend("b200").hermitian_rank_k_update(acc, pkg.ComplexDense.from_array(a),
                                                    pkg.FlopLedger())
    got = acc.matrix.array
    assert np.all(np.isnan(got[iu]))
    exp = np.tril(c0 + a.conj().T @ a)
    assert rel_fro(np.tril(got), exp) <= 1e-14


def test_her2k_and_strided_views(pkg):
    rng = np.random.default_rng(3)
    big = pkg.ComplexDense.zeros(40, 70, capacity_rows=64)
    big.array[:] = rand_complex(rng, 40, 70)
    x = big.block(3, 21)
    b = pkg.ComplexDense.from_array(rand_complex(rng, 21, 70))
    acc = pkg.HermitianAccumulator(70)
    led = pkg.FlopLedger()
    pkg.get_backend().hermitian_rank_2k_update(acc, x, b, led)
    exp = np.tril(x.array.conj().T @ b.array + b.array.conj().T @ x.array)
    assert rel_fro(np.tril(acc.matrix.array), exp) <= 1e-14
    assert led.hermitian_rank_2k == 8 * 21 * 70 * 70


@pytest.mark.parametrize("conj", [False, True])
def test_gemm_alpha_beta(pkg, conj):
    rng = np.random.default_rng(5)
    m, n, k = 70, 45, 33
    a = rand_complex(rng, k, m) if conj else rand_complex(rng, m, k)
    b = rand_complex(rng, k, n)
    c0 = rand_complex(rng, m, n)
    c = pkg.ComplexDense.from_array(c0)
    al, be = 2.0 + 1.0j, 0.5 - 0.25j
    pkg.get_backend().general_product(c, pkg.ComplexDense.from_array(a),
                                      pkg.ComplexDense.from_array(b), conj, al, be,
                                      pkg.FlopLedger())
    op = a.conj().T if conj else a
    assert rel_fro(c.array, al * (op @ b) + be * c0) <= 1e-14


def test_hemm_reads_lower_only_and_trmm(pkg):
    rng = np.random.default_rng(9)
    t_full = hermitian_from_lower(rand_complex(rng, 9, 9))
    t_st = t_full.copy()
    t_st[np.triu_indices(9, 1)] = np.nan
    t_st[np.diag_indices(9)] += 5j  # imaginary diagonal is ignored
    a = rand_complex(rng, 9, 77)
    x = pkg.ComplexDense.from_array(rand_complex(rng, 9, 77))
    x0 = x.array.copy()
    pkg.get_backend().hermitian_product(x, pkg.ComplexDense.from_array(t_st),
                                        pkg.ComplexDense.from_array(a), True, 0.5,
                                        pkg.FlopLedger())
    assert rel_fro(x.array, 0.5 * t_full @ a + x0) <= 1e-14
    low = np.tril(rand_complex(rng, 9, 9))
    st = low.copy()
    st[np.triu_indices(9, 1)] = np.nan
    for conj in (False, True):
        y = pkg.ComplexDense.zeros(9, 77)
        pkg.get_backend().triangular_product(y, pkg.ComplexDense.from_array(st),
                                             pkg.ComplexDense.from_array(a), conj,
                                             pkg.FlopLedger())
        op = low.conj().T if conj else low
        assert rel_fro(y.array, op @ a) <= 1e-14


def test_cholesky_contract(pkg):
    be = pkg.get_backend()
    rng = np.random.default_rng(11)
    g = rand_complex(rng, 81, 81)
    t = g @ g.conj().T / 81 + np.eye(81)
    led = pkg.FlopLedger()
    c = be.cholesky_factor(pkg.ComplexDense.from_array(t), led)
    assert rel_fro(c.array @ c.array.conj().T, t) <= 1e-14
    assert np.all(np.triu(c.array, 1) == 0)
    assert led.cholesky == 4 * 81**3 // 3
    with pytest.raises(pkg.NotHPDError) as e:
        be.cholesky_factor(pkg.ComplexDense.from_array(np.diag([1.0, 2.0, -3.0, 4.0]) + 0j), led)
    assert e.value.pivot == 2
    bad = np.eye(3, dtype=complex)
    bad[1, 0] = np.nan
    with pytest.raises(pkg.ContractViolationError):
        be.cholesky_factor(pkg.ComplexDense.from_array(bad), led)


def test_mirror_and_scale_rows(pkg):
    rng = np.random.default_rng(2)
    acc = pkg.HermitianAccumulator(75)
    acc.matrix.array[:] = rand_complex(rng, 75, 75)
    low = acc.matrix.array.copy()
    full = acc.mirror_to_full().array
    np.testing.assert_array_equal(full, full.conj().T)
    np.testing.assert_array_equal(np.tril(full, -1), np.tril(low, -1))
    np.testing.assert_array_equal(full.diagonal().imag, 0)
    b = pkg.ComplexDense.from_array(rand_complex(rng, 13, 20))
    b0 = b.array.copy()
    d = rng.uniform(0.1, 2, 13)
    pkg.scale_rows(b, d, pkg.FlopLedger())
    np.testing.assert_array_equal(b.array, b0 * d[:, None])
    acc = pkg.HermitianAccumulator(3)
    acc.matrix.array[2, 1] = np.inf
    with pytest.raises(pkg.ContractViolationError):
        acc.mirror_to_full()


# ---------------------------------------------------------------- A/B generation

def test_compute_ab_small_vs_reference_golden(pkg):
    d = golden("ab_small.npz")
    c = pkg.compute_AB(spec_from_golden(d))
    assert rel_fro(c.A_star.array, d["A"]) <= 1e-13
    assert rel_fro(c.B_star.array, d["B"]) <= 1e-13
    np.testing.assert_array_equal(c.udot_norms, d["udot_norms"])
    assert c.A_star.leading_dimension == c.layout.capacity_rows


def test_compute_ab_high_l_vs_reference_golden(pkg):
    """l_sph 12, 14 (HSDLA_MAX_LSPH), 13 with x = |K| r up to ~21: every Bessel regime at
    high order; checked per (atom, l) block so no block hides behind larger ones."""
    d = golden("ab_high.npz")
    c = pkg.compute_AB(spec_from_golden(d))
    a, b = c.A_star.array, c.B_star.array
    assert rel_fro(a, d["A"]) <= 1e-13
    assert rel_fro(b, d["B"]) <= 1e-13
    r0 = 0
    for l_max in d["spec_l_sph"]:
        for l in range(int(l_max) + 1):
            rows = slice(r0 + l * l, r0 + (l + 1) ** 2)
            assert rel_fro(a[rows], d["A"][rows]) <= 1e-12, (l_max, l)
            assert rel_fro(b[rows], d["B"][rows]) <= 1e-12, (l_max, l)
        r0 += (int(l_max) + 1) ** 2


def test_compute_ab_c1_vs_reference_golden(pkg):
    from paper_1602_06589_b200 import configs

    d = golden("ab_c1.npz")
    c = pkg.compute_AB(configs.make_instance("C1").spec)
    a, b = c.A_star.array, c.B_star.array
    assert rel_fro(a[:, d["cols"]], d["A_cols"]) <= 1e-13
    assert rel_fro(b[:, d["cols"]], d["B_cols"]) <= 1e-13
    assert rel_fro(a @ d["V"], d["AV"]) <= 1e-13
    # per (atom, l) block errors: small-Wronskian rows must not hide errors elsewhere
    ref_a = of.compute_ab(configs.make_instance("C1").spec)[0]
    for r0 in range(0, a.shape[0], 7):
        assert rel_fro(a[r0:r0 + 7], ref_a[r0:r0 + 7]) <= 1e-12


# ---------------------------------------------------------------- builds

@pytest.mark.parametrize("ci", range(7))
def test_build_all_small_vs_reference_golden(pkg, ci):
    c = build_case(golden("build_small.npz"), ci)
    heights = c["heights"]
    lay = pkg.AtomBlockLayout(tuple(heights), c["cap"])
    r = sum(heights)
    a = pkg.ComplexDense.zeros(r, c["A"].shape[1], capacity_rows=lay.capacity_rows)
    b = pkg.ComplexDense.zeros(r, c["A"].shape[1], capacity_rows=lay.capacity_rows)
    a.array[:] = c["A"]
    b.array[:] = c["B"]
    coeffs = pkg.StackedCoefficients(a, b, lay, c["udot"])
    cd = pkg.ComplexDense.from_array
    tm = pkg.TMatrixSet([cd(t) for t in c["t_aa"]], [cd(t) for t in c["t_ab"]],
                        [cd(t) for t in c["t_bb"]], [0] * len(heights), [0] * len(heights))
    h, s, rep = pkg.build_all(coeffs, tm, pkg.BuildConfig(force_general_path=c["force"]))
    assert rel_fro(h.array, c["H"]) <= TOL
    assert rel_fro(s.array, c["S"]) <= TOL
    np.testing.assert_array_equal(h.array, h.array.conj().T)
    np.testing.assert_array_equal(s.array, s.array.conj().T)
    assert [rep.ledger.as_dict()[k] for k in LEDGER_KEYS] == list(c["ledger"])
    assert rep.hpd_mask == c["mask"]


def _c1_gpu(pkg):
    from paper_1602_06589_b200 import configs

    inst = configs.make_instance("C1")
    coeffs = pkg.compute_AB(inst.spec)
    return pkg.build_all(coeffs, inst.tmats, pkg.BuildConfig())


def test_c1_end_to_end_vs_reference_golden(pkg):
    d = golden("build_c1.npz")
    h, s, rep = _c1_gpu(pkg)
    hh, ss = h.array, s.array
    assert rel_fro(hh @ d["V"], d["HV"]) <= TOL
    assert rel_fro(ss @ d["V"], d["SV"]) <= TOL
    assert rel_fro(np.diag(hh), d["H_diag"]) <= TOL
    assert rel_fro(hh[:, 0], d["H_col0"]) <= TOL
    assert abs(np.linalg.norm(hh) - d["H_fro"]) <= TOL * d["H_fro"]
    assert abs(np.linalg.norm(ss) - d["S_fro"]) <= TOL * d["S_fro"]
    assert [rep.ledger.as_dict()[k] for k in LEDGER_KEYS] == list(d["ledger"])


def test_c2_end_to_end_vs_oracle(pkg):
    from paper_1602_06589_b200 import configs

    inst = configs.make_instance("C2")
    a, b, norms, offs = of.compute_ab(inst.spec)
    tm = inst.tmats
    heights = list(np.diff(offs))
    h_o, s_o, led, mask = ob.build_all(a, b, norms, heights, [t.array for t in tm.t_aa],
                                       [t.array for t in tm.t_ab], [t.array for t in tm.t_bb])
    coeffs = pkg.compute_AB(inst.spec)
    assert rel_fro(coeffs.A_star.array, a) <= 1e-13
    assert rel_fro(coeffs.B_star.array, b) <= 1e-13
    h, s, rep = pkg.build_all(coeffs, tm, pkg.BuildConfig())
    assert rel_fro(h.array, h_o) <= TOL
    assert rel_fro(s.array, s_o) <= TOL
    assert rep.hpd_mask == mask
    assert rep.ledger == pkg.predict_flops(len(heights), heights, inst.spec.n_basis, mask)


def test_device_pipeline_matches_drop_in(pkg):
    """HSPipeline (A/B generated in HBM, B scaled in the producer) == compute_AB + build_all.
    The two paths cut the stream-K work differently (the drop-in copies column ranges to the
    host as they finish), so agreement is to rounding, not bitwise."""
    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats

    inst = configs.make_instance("C1")
    h_ref, s_ref, _ = _c1_gpu(pkg)
    dspec = DeviceSpec(inst.spec)
    pipe = HSPipeline(inst.spec.n_basis, dspec.heights)
    res = pipe.run(dspec, pack_tmats(inst.tmats))
    n = inst.spec.n_basis
    h = pipe.H[:n, :n].cpu().numpy().T
    s = pipe.S[:n, :n].cpu().numpy().T
    assert rel_fro(h, h_ref.array) <= 1e-14
    assert rel_fro(s, s_ref.array) <= 1e-14
    np.testing.assert_array_equal(h, h.conj().T)
    assert all(res["hpd_mask"])


def test_backup_invariance_bitwise(pkg):
    c = build_case(golden("build_small.npz"), 1)
    heights = c["heights"]
    lay = pkg.AtomBlockLayout(tuple(heights), c["cap"])

    def coeffs():
        r = sum(heights)
        a = pkg.ComplexDense.zeros(r, c["A"].shape[1], capacity_rows=lay.capacity_rows)
        b = pkg.ComplexDense.zeros(r, c["A"].shape[1], capacity_rows=lay.capacity_rows)
        a.array[:] = c["A"]
        b.array[:] = c["B"]
        return pkg.StackedCoefficients(a, b, lay, c["udot"])

    cd = pkg.ComplexDense.from_array
    tm = pkg.TMatrixSet([cd(t) for t in c["t_aa"]], [cd(t) for t in c["t_ab"]],
                        [cd(t) for t in c["t_bb"]], [0, 0], [0, 0])
    calls = []

    def regen(co):
        calls.append(1)
        co.A_star.array[:] = c["A"]
        co.B_star.array[:] = c["B"]

    h1, s1, _ = pkg.build_all(coeffs(), tm, pkg.BuildConfig(backup=True))
    h2, s2, _ = pkg.build_all(coeffs(), tm, pkg.BuildConfig(backup=False), regenerate=regen)
    np.testing.assert_array_equal(h1.array, h2.array)
    np.testing.assert_array_equal(s1.array, s2.array)
    assert calls == [1]


def test_build_hs_overlapped_host_copy_matches_device(pkg):
    """build_hs copies H, S to pinned host memory in column ranges overlapped with the
    compute; the host result matches the device-only run and the reference golden, and
    repeated calls are bitwise identical."""
    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, build_hs, pack_tmats

    inst = configs.make_instance("C1")
    h, s, res = build_hs(inst.spec, inst.tmats)
    dspec = DeviceSpec(inst.spec)
    pipe = HSPipeline(inst.spec.n_basis, dspec.heights)
    pipe.run(dspec, pack_tmats(inst.tmats))
    hd, sd = (m.cpu().numpy().T for m in pipe.result_views())
    assert rel_fro(h.array, hd) <= 1e-14 and rel_fro(s.array, sd) <= 1e-14
    h2, s2, _ = build_hs(inst.spec, inst.tmats)
    np.testing.assert_array_equal(h.array, h2.array)
    np.testing.assert_array_equal(s.array, s2.array)
    d = golden("build_c1.npz")
    assert rel_fro(h.array @ d["V"], d["HV"]) <= TOL
    assert res["d2h_bytes"] == 2 * 16 * inst.spec.n_basis ** 2


def test_build_hs_many_pipelined_kpoints_match_single_calls(pkg):
    """A k-point batch through the pipelined path (copies of k-point i overlap the compute
    of i+1, varying N_G per k-point) equals per-k-point synchronous calls and the oracle."""
    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.pipeline import build_hs, build_hs_many

    inst = configs.make_instance("C1")
    specs = [configs.kpoint_variant(inst, i) for i in range(4)]
    assert len({s.n_basis for s in specs}) > 1  # different G-sets per k-point
    seen = []

    def on_result(i, h, s, res):
        h1, s1, _ = build_hs(specs[i], inst.tmats)
        assert rel_fro(h.array, h1.array) <= 1e-14 and rel_fro(s.array, s1.array) <= 1e-14
        seen.append((i, h.array.copy(), s.array.copy()))

    build_hs_many(specs, inst.tmats, on_result=on_result)
    assert [i for i, _, _ in seen] == [0, 1, 2, 3]
    i, h, s = seen[2]
    a, b, norms, offs = of.compute_ab(specs[2])
    tm = inst.tmats
    h_o, s_o, _, _ = ob.build_all(a, b, norms, list(np.diff(offs)), [t.array for t in tm.t_aa],
                                  [t.array for t in tm.t_ab], [t.array for t in tm.t_bb])
    assert rel_fro(h, h_o) <= TOL and rel_fro(s, s_o) <= TOL
