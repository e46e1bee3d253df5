"""Edge shapes of the composed build and compute_AB on the GPU, against the oracle
(which is pinned to the reference's goldens): tile and K-chunk boundaries (N_G and block
heights at 1, 15/16/17, 63/64/65), single atoms, l = 0 blocks, T smaller than its block,
mixed HPD, a K = 0 vector, and k-point batches whose N_G varies."""
import numpy as np
import pytest

from conftest import rand_complex, rel_fro
from oracle import build as ob
from oracle import flapw as of

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


def _case(pkg, seed, heights, n_g, t_sizes=None, shifts=None):
    rng = np.random.default_rng(seed)
    lay = pkg.AtomBlockLayout(tuple(heights))
    r = lay.total_rows
    a = pkg.ComplexDense.zeros(r, n_g, capacity_rows=lay.capacity_rows)
    b = pkg.ComplexDense.zeros(r, n_g, capacity_rows=lay.capacity_rows)
    a.array[:] = rand_complex(rng, r, n_g)
    b.array[:] = rand_complex(rng, r, n_g)
    u = rng.uniform(0.2, 1.5, r)
    co = pkg.StackedCoefficients(a, b, lay, u)
    t_sizes = t_sizes or list(heights)
    shifts = shifts or [2.0] * len(heights)
    taa = [_hermitian(rng, m, s) for m, s in zip(t_sizes, shifts)]
    tbb = [_hermitian(rng, m, 1.0) for m in t_sizes]
    tab = [rand_complex(rng, m, m) / m for m in t_sizes]
    cd = pkg.ComplexDense.from_array
    tm = pkg.TMatrixSet([cd(t) for t in taa], [cd(t) for t in tab], [cd(t) for t in tbb],
                        [0] * len(heights), [0] * len(heights))
    return co, tm, (a.array.copy(), b.array.copy(), u.copy(), taa, tab, tbb)


@pytest.mark.parametrize("heights,n_g", [((1,), 1), ((1,), 2), ((4,), 63), ((4,), 64), ((4,), 65),
                                         ((16,), 17), ((15, 17), 129), ((1, 64, 3), 64),
                                         ((9, 9, 9, 9, 9, 9, 9), 200)])
def test_build_all_edge_shapes(pkg, heights, n_g):
    co, tm, (a, b, u, taa, tab, tbb) = _case(pkg, sum(heights) * 7 + n_g, heights, n_g)
    h, s, rep = pkg.build_all(co, tm, pkg.BuildConfig())
    want = ob.build_all(a, b, u, list(heights), taa, tab, tbb)
    assert rel_fro(s.array, want[1]) <= TOL
    assert rel_fro(h.array, want[0]) <= TOL
    np.testing.assert_array_equal(h.array, h.array.conj().T)
    np.testing.assert_array_equal(s.array, s.array.conj().T)
    assert rep.hpd_mask == list(want[3])


def test_build_all_small_t_and_non_hpd(pkg):
    """T smaller than its block (rows beyond m contribute nothing) and a non-HPD T_AA next
    to HPD ones (device-side branch selection)."""
    heights = (16, 9, 25)
    co, tm, (a, b, u, taa, tab, tbb) = _case(pkg, 5, heights, 97, t_sizes=[9, 9, 16],
                                             shifts=[2.0, -2.0, 2.0])
    h, s, rep = pkg.build_all(co, tm, pkg.BuildConfig())
    want = ob.build_all(a, b, u, list(heights), taa, tab, tbb)
    assert rel_fro(h.array, want[0]) <= TOL and rel_fro(s.array, want[1]) <= TOL
    assert rep.hpd_mask == [True, False, True] == list(want[3])


def test_compute_ab_single_atom_l0_and_zero_k(pkg):
    from paper_1602_06589_b200 import RadialBoundaryData, SystemSpec

    rng = np.random.default_rng(4)
    kv = rng.standard_normal((5, 3))
    kv[0] = 0.0
    rad = [RadialBoundaryData(u=np.array([0.5]), u_prime=np.array([0.7]), udot=np.array([0.3]),
                              udot_prime=np.array([0.9]), energy=np.zeros(1),
                              udot_norm=np.array([0.2]))]
    spec = SystemSpec(positions=np.zeros((1, 3)), rotations=np.eye(3)[None], mt_radius=np.array([2.0]),
                      l_sph=np.array([0]), l_nonsph=np.array([0]), k_point=np.zeros(3),
                      k_vectors=kv, omega=100.0, radial=rad)
    c = pkg.compute_AB(spec)
    a, b, norms, _ = of.compute_ab(spec)
    assert c.A_star.rows == 1 and c.n_basis == 5
    assert rel_fro(c.A_star.array, a) <= 1e-14 and rel_fro(c.B_star.array, b) <= 1e-14
    np.testing.assert_array_equal(c.udot_norms, norms)


def test_kpoint_batch_with_varying_basis_sizes(pkg):
    """build_hs_many over k-points whose G-sets differ in size (one pipeline sized to the
    largest), each result equal to its own single build."""
    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.pipeline import build_hs, build_hs_many

    inst = configs.make_instance("C1")
    specs = [configs.kpoint_variant(inst, r) for r in range(3)]
    assert len({s.n_basis for s in specs}) > 1
    got = {}
    build_hs_many(specs, inst.tmats, on_result=lambda i, h, s, r: got.__setitem__(
        i, (h.array.copy(), s.array.copy())))
    for i, sp in enumerate(specs):
        h, s, _ = build_hs(sp, inst.tmats)
        assert got[i][0].shape == (sp.n_basis, sp.n_basis)
        assert rel_fro(got[i][0], h.array) <= 1e-14 and rel_fro(got[i][1], s.array) <= 1e-14


def test_async_builds_three_in_flight_out_of_order(pkg):
    """hsdla_setup_hs_async with three k-points in flight (the oldest is completed into the
    stash when the third is enqueued) and finished out of order; each host result equals a
    synchronous build, and a finished ticket cannot be finished twice."""
    import torch

    from paper_1602_06589_b200 import NativeLibraryError, configs
    from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, build_hs, pack_tmats

    inst = configs.make_instance("C1")
    specs = [configs.kpoint_variant(inst, r) for r in range(3)]
    n_cap = max(s.n_basis for s in specs)
    tp = pack_tmats(inst.tmats)
    pipe = HSPipeline(n_cap, DeviceSpec(specs[0]).heights)
    outs = [(torch.empty((s.n_basis, s.n_basis), dtype=torch.complex128, pin_memory=True),
             torch.empty((s.n_basis, s.n_basis), dtype=torch.complex128, pin_memory=True))
            for s in specs]
    tickets = [pipe.run_async(DeviceSpec(s), tp, host_out=o) for s, o in zip(specs, outs)]
    for k in (2, 0, 1):
        res = pipe.finish(tickets[k])
        assert res["hpd_mask"] == [True] * specs[k].n_atoms
    for s, (h, sm) in zip(specs, outs):
        h1, s1, _ = build_hs(s, inst.tmats)
        assert rel_fro(h.numpy().T, h1.array) <= 1e-14 and rel_fro(sm.numpy().T, s1.array) <= 1e-14
    with pytest.raises((NativeLibraryError, KeyError)):
        pipe.finish(tickets[0])


def test_build_all_host_sourced_upload(pkg, monkeypatch):
    """compute_AB's pinned stacks uploaded by the native build itself (B overlapped with the
    A-part of S, S accumulated in two launches; used for large stacks): same H, S as the
    default upload path to rounding and the oracle to 1e-12, and exactly Hermitian."""
    from paper_1602_06589_b200 import builder, configs, device

    inst = configs.make_instance("C1")
    co = pkg.compute_AB(inst.spec)
    assert device.pinned_sources(co.A_star, co.B_star) is not None
    h0, s0, r0 = pkg.build_all(co, inst.tmats, pkg.BuildConfig())
    monkeypatch.setattr(builder, "HOST_SOURCED_MIN_BYTES", 0)
    co = pkg.compute_AB(inst.spec)
    h1, s1, r1 = pkg.build_all(co, inst.tmats, pkg.BuildConfig())
    assert rel_fro(h1.array, h0.array) <= 1e-14 and rel_fro(s1.array, s0.array) <= 1e-14
    a, b, norms, offs = of.compute_ab(inst.spec)
    tm = inst.tmats
    h_o, s_o, _, mask = ob.build_all(a, b, norms, list(np.diff(offs)), [t.array for t in tm.t_aa],
                                     [t.array for t in tm.t_ab], [t.array for t in tm.t_bb])
    assert rel_fro(h1.array, h_o) <= TOL and rel_fro(s1.array, s_o) <= TOL
    np.testing.assert_array_equal(s1.array, s1.array.conj().T)
    assert r1.hpd_mask == r0.hpd_mask == list(mask)
    # a window that is not at the top of its allocation is not host-sourced
    assert device.pinned_sources(co.A_star.block(1, co.A_star.rows - 1), co.B_star) is None


def _spec_variant(pkg, spec, rotations=None, l_sph=None):
    return pkg.SystemSpec(positions=spec.positions,
                          rotations=spec.rotations if rotations is None else rotations,
                          mt_radius=spec.mt_radius, l_sph=spec.l_sph if l_sph is None else l_sph,
                          l_nonsph=spec.l_nonsph if l_sph is None else l_sph, k_point=spec.k_point,
                          k_vectors=spec.k_vectors, omega=spec.omega, radial=spec.radial)


@pytest.mark.parametrize("variant", ["types", "rotated", "reference_forms", "single_atom_types"])
def test_template_path_variants_vs_oracle(pkg, variant):
    """The device pipeline's per-type template path (hsdla_build_args.atom_type) and its
    fallbacks against the oracle: BASELINE-style shared types; every atom rotated differently
    (one type per atom); the reference H forms (templates for A / UB, per-atom T applications
    on B); a one-atom-per-type system."""
    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats

    inst = configs.make_instance("C1")
    spec, tm = inst.spec, inst.tmats
    if variant == "rotated":
        rng = np.random.default_rng(4)
        rots = np.array([np.linalg.qr(rng.standard_normal((3, 3)))[0] for _ in range(spec.n_atoms)])
        spec = _spec_variant(pkg, spec, rotations=rots)
    if variant == "single_atom_types":
        cd = pkg.ComplexDense.from_array
        tm = pkg.TMatrixSet([cd(t.array.copy()) for t in tm.t_aa], [cd(t.array.copy()) for t in tm.t_ab],
                            [cd(t.array.copy()) for t in tm.t_bb], list(tm.l_sph), list(tm.l_nonsph))
    dspec = DeviceSpec(spec)
    pipe = HSPipeline(spec.n_basis, dspec.heights, h_reference_form=(variant == "reference_forms"))
    res = pipe.run(dspec, pack_tmats(tm))
    want_types = {"types": 2, "rotated": 4, "reference_forms": 2, "single_atom_types": 4}[variant]
    assert res["template_types"] == want_types
    assert all(res["joint_t"]) == (variant != "reference_forms")
    h_t, s_t = pipe.result_views()
    h, s = h_t.cpu().numpy().T, s_t.cpu().numpy().T
    a, b, norms, offs = of.compute_ab(spec)
    h_o, s_o, _, mask = ob.build_all(a, b, norms, list(np.diff(offs)), [t.array for t in tm.t_aa],
                                     [t.array for t in tm.t_ab], [t.array for t in tm.t_bb])
    assert res["hpd_mask"] == list(mask)
    assert rel_fro(h, h_o) <= TOL and rel_fro(s, s_o) <= TOL
    np.testing.assert_array_equal(h, h.conj().T)
    # the reused T preparation (second k-point of a batch: B not written on the joint path)
    res2 = pipe.run(dspec, pack_tmats(tm))
    h2 = pipe.result_views()[0].cpu().numpy().T
    np.testing.assert_array_equal(h2, h)
    assert res2["template_types"] == want_types


def test_template_path_off_for_short_t(pkg):
    """T smaller than its block: the per-atom path (template_types = 0), still exact."""
    from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats
    from paper_1602_06589_b200 import configs

    inst = configs.make_instance("C1")
    spec = inst.spec
    cd = pkg.ComplexDense.from_array
    m = 36  # (l = 5)^2 < 49 rows of every block
    tm = pkg.TMatrixSet([cd(t.array[:m, :m].copy()) for t in inst.tmats.t_aa],
                        [cd(t.array[:m, :m].copy()) for t in inst.tmats.t_ab],
                        [cd(t.array[:m, :m].copy()) for t in inst.tmats.t_bb],
                        list(inst.tmats.l_sph), list(inst.tmats.l_nonsph))
    dspec = DeviceSpec(spec)
    pipe = HSPipeline(spec.n_basis, dspec.heights)
    res = pipe.run(dspec, pack_tmats(tm))
    assert res["template_types"] == 0
    h_t, s_t = pipe.result_views()
    a, b, norms, offs = of.compute_ab(spec)
    h_o, s_o, _, _ = ob.build_all(a, b, norms, list(np.diff(offs)), [t.array for t in tm.t_aa],
                                  [t.array for t in tm.t_ab], [t.array for t in tm.t_bb])
    assert rel_fro(h_t.cpu().numpy().T, h_o) <= TOL and rel_fro(s_t.cpu().numpy().T, s_o) <= TOL


def test_template_path_mixed_l_types(pkg):
    """Types with different l_sph (block heights 25 and 49) and a lone atom of a third type: the
    template generator runs per l group, the expansion per atom height; vs the oracle, and a
    batch k-point reusing the T preparation (B not rewritten) equals the first bitwise."""
    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats

    base = configs.make_instance("C1").spec
    rng = np.random.default_rng(17)
    l_sph = np.array([4, 4, 6, 6, 2])
    n_at = len(l_sph)
    pos = rng.uniform(0, 8.0, (n_at, 3))
    rad = []
    for l in (4, 6, 2):
        n = l + 1
        rad.append(pkg.RadialBoundaryData(u=rng.uniform(0.1, 1, n), u_prime=rng.uniform(0.1, 1, n),
                                          udot=rng.uniform(0.1, 1, n), udot_prime=rng.uniform(0.1, 1, n),
                                          energy=np.zeros(n), udot_norm=np.sqrt(rng.uniform(0.01, 0.1, n))))
    radial = [rad[0], rad[0], rad[1], rad[1], rad[2]]
    spec = pkg.SystemSpec(positions=pos, rotations=np.tile(np.eye(3), (n_at, 1, 1)),
                          mt_radius=np.array([2.0, 2.0, 2.2, 2.2, 1.8]), l_sph=l_sph, l_nonsph=l_sph,
                          k_point=base.k_point, k_vectors=base.k_vectors, omega=base.omega,
                          radial=radial)
    cd = pkg.ComplexDense.from_array
    ts = {}
    for l in (4, 6, 2):
        m = (l + 1) ** 2
        ts[l] = tuple(cd(x) for x in (_hermitian(rng, m, 2.0), rand_complex(rng, m, m) / m,
                                      _hermitian(rng, m, 2.0)))
    tm = pkg.TMatrixSet([ts[l][0] for l in l_sph], [ts[l][1] for l in l_sph],
                        [ts[l][2] for l in l_sph], list(l_sph), list(l_sph))
    dspec = DeviceSpec(spec)
    pipe = HSPipeline(spec.n_basis, dspec.heights)
    tp = pack_tmats(tm)
    res = pipe.run(dspec, tp)
    assert res["template_types"] == 3 and all(res["joint_t"])
    h_t, s_t = pipe.result_views()
    h, s = h_t.cpu().numpy().T, s_t.cpu().numpy().T
    a, b, norms, offs = of.compute_ab(spec)
    h_o, s_o, _, _ = ob.build_all(a, b, norms, list(np.diff(offs)), [t.array for t in tm.t_aa],
                                  [t.array for t in tm.t_ab], [t.array for t in tm.t_bb])
    assert rel_fro(h, h_o) <= TOL and rel_fro(s, s_o) <= TOL
    pipe.run(dspec, tp)
    h2_t, s2_t = pipe.result_views()
    np.testing.assert_array_equal(h2_t.cpu().numpy().T, h)
    np.testing.assert_array_equal(s2_t.cpu().numpy().T, s)
