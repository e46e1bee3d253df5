"""CPU-only tests: storage types, closed forms, ledger replica, config generator, the
C ABI's exported symbols, and the fail-loudly contract without a GPU."""
import os
import re

import numpy as np
import pytest

from conftest import LEDGER_KEYS, REPO, build_case, golden
import paper_1602_06589_b200 as pkg
from paper_1602_06589_b200 import configs


# -- storage (reference matrix.py:21-194, tests/test_matrix_core.py) ----------------

def test_complex_dense_views_share_memory_and_ld():
    m = pkg.ComplexDense.zeros(7, 4, capacity_rows=12)
    assert m.leading_dimension == 12 and m.base.flags.f_contiguous
    assert pkg.ComplexDense.zeros(5, 3).array.flags.f_contiguous
    blk = m.block(2, 3)
    blk.array[:] = 1 + 2j
    np.testing.assert_array_equal(m.array[2:5], np.full((3, 4), 1 + 2j))
    assert blk.shares_buffer(m) and m.full_capacity().rows == 12
    with pytest.raises(pkg.ContractViolationError):
        m.block(6, 2)
    with pytest.raises(pkg.ContractViolationError):
        pkg.ComplexDense.zeros(5, 2, capacity_rows=3)
    with pytest.raises(pkg.ContractViolationError):
        pkg.ComplexDense(np.zeros((2, 2)))  # not complex128
    f = pkg.ComplexDense.from_array([[1 + 0j, 3], [2, 4]])
    np.testing.assert_array_equal(np.asarray(f.array).ravel(order="F"), [1, 2, 3, 4])


def test_layout_and_ledger():
    lay = pkg.AtomBlockLayout((4, 9, 1), 9)
    np.testing.assert_array_equal(lay.offsets, [0, 4, 13, 14])
    assert lay.total_rows == 14 and lay.capacity_rows == 27
    for bad in ((0, 3), ()):
        with pytest.raises(pkg.ContractViolationError):
            pkg.AtomBlockLayout(bad)
    with pytest.raises(pkg.ContractViolationError):
        pkg.AtomBlockLayout((4, 9), 4)
    led = pkg.FlopLedger()
    led.add("hermitian_rank_k", 10)
    led.add("cholesky", 5)
    assert led.total == 15 and led.as_dict()["total"] == 15
    with pytest.raises(pkg.ContractViolationError):
        led.add("row_scale", -1)


def test_stacked_coefficients_validation():
    lay = pkg.AtomBlockLayout((4,))
    with pytest.raises(pkg.ContractViolationError):
        pkg.StackedCoefficients(pkg.ComplexDense.zeros(3, 5), pkg.ComplexDense.zeros(4, 5), lay,
                                np.ones(4))
    with pytest.raises(pkg.ContractViolationError):
        pkg.StackedCoefficients(pkg.ComplexDense.zeros(4, 5), pkg.ComplexDense.zeros(4, 5), lay,
                                np.ones(3))


# -- closed forms (reference builder.py:318-385, tests/test_builder.py:371-439) ------

def test_estimate_memory_paper_examples():
    assert pkg.estimate_memory(512, 49, 2256, backup=True) == 3_703_738_368
    assert pkg.estimate_memory(384, 81, 29144, backup=True) == 71_605_642_240
    assert pkg.estimate_memory(1, 1, 1, backup=False) == 64
    assert pkg.estimate_memory(3, 4, 5, backup=False) == 32 * 3 * 4 * 5 + 32 * 25
    with pytest.raises(OverflowError):
        pkg.estimate_memory(2**30, 2**20, 2**30, backup=True)
    with pytest.raises(pkg.ContractViolationError):
        pkg.estimate_memory(0, 1, 1, backup=False)


def test_predict_flops_hand_totals():
    led = pkg.predict_flops(1, [1], 1, [True])
    assert (led.hermitian_rank_k, led.row_scale, led.general_product, led.hermitian_product,
            led.hermitian_rank_2k, led.cholesky, led.triangular_product) == (12, 2, 8, 8, 8, 1, 4)
    led = pkg.predict_flops(1, [1], 1, [False])
    assert led.cholesky == 0 and led.hermitian_product == 16 and led.general_product == 16


def test_large_update_fraction_paper_targets():
    f1 = pkg.large_update_fraction(512, [49] * 512, 2256, [True] * 256 + [False] * 256)
    assert abs(f1 * 100 - 98.06) <= 0.5
    f2 = pkg.large_update_fraction(384, [81] * 384, 29144, [True] * 192 + [False] * 192)
    assert abs(f2 * 100 - 99.75) <= 0.5


@pytest.mark.parametrize("ci", range(7))
def test_build_ledger_replicates_reference_ledger(ci):
    c = build_case(golden("build_small.npz"), ci)
    sizes = [t.shape[0] for t in c["t_aa"]]
    led = pkg.build_ledger(c["heights"], sizes, c["A"].shape[1], c["mask"], c["force"])
    assert [led.as_dict()[k] for k in LEDGER_KEYS] == list(c["ledger"])


def test_build_ledger_equals_predict_flops_when_t_matches_blocks():
    heights = [49, 49, 81]
    mask = [True, False, True]
    assert pkg.build_ledger(heights, heights, 600, mask, False) == \
        pkg.predict_flops(3, heights, 600, mask)


# -- configuration generator ---------------------------------------------

@pytest.mark.parametrize("name,target,rows", [("C1", 600, 196), ("C2", 3000, 1296),
                                              ("C3", 8000, 5184), ("C4", 13000, 13068),
                                              ("C5", 5000, 2592)])
def test_configs_sizes(name, target, rows):
    inst = configs.make_instance(name, n_kpoints=1)
    spec = inst.spec
    assert abs(spec.n_basis - target) <= 0.02 * target
    assert sum((int(l) + 1) ** 2 for l in spec.l_sph) == rows
    norms = np.linalg.norm(spec.k_vectors, axis=1)
    assert np.all(np.diff(norms) >= -1e-12)  # sorted by |K|


def test_configs_deterministic_and_t_hpd():
    a = configs.make_instance("C1")
    b = configs.make_instance("C1")
    np.testing.assert_array_equal(a.spec.k_vectors, b.spec.k_vectors)
    np.testing.assert_array_equal(a.tmats.t_aa[0].array, b.tmats.t_aa[0].array)
    for t in a.tmats.t_aa:
        assert np.linalg.eigvalsh(t.array)[0] > 1.5  # always HPD
    assert a.tmats.t_aa[0] is a.tmats.t_aa[1]  # atoms of a type share T objects
    c5 = configs.make_instance("C5")
    assert len(c5.specs) == 64
    k = np.array([s.k_point for s in c5.specs])
    b_ = 2 * np.pi / 14.0
    assert np.all(k[:, 0] >= k[:, 1]) and np.all(k[:, 1] >= k[:, 2]) and np.all(k >= 0)
    assert np.all(k <= 0.5 * b_ + 1e-12)
    v = configs.kpoint_variant(a, 3)
    assert v.n_atoms == a.spec.n_atoms and not np.allclose(v.k_point, a.spec.k_point)


# -- C ABI ----------------------------------------------------------------------------

def test_library_exports_every_declared_symbol():
    with open(os.path.join(REPO, "include", "hsdla_b200.h")) as f:
        header = f.read()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(hsdla_\w+)\(", header, re.M))
    assert len(declared) >= 17
    lib = pkg._native.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(pkg._native.SIGNATURES)
    assert lib.hsdla_version() == 1
    assert lib.hsdla_complex_mul_products() in (3, 4)
    # panel ownership: balanced pairs j <-> nb-1-j
    own = [lib.hsdla_panel_owner(10, 3, j) for j in range(10)]
    assert own == [0, 1, 2, 0, 1, 1, 0, 2, 1, 0]


def test_gpu_entry_points_fail_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    inst = configs.make_instance("C1")
    with pytest.raises(pkg.NativeLibraryError):
        pkg.compute_AB(inst.spec)
    acc = pkg.HermitianAccumulator(3)
    with pytest.raises(pkg.NativeLibraryError):
        acc.mirror_to_full()


def test_configuration_errors():
    with pytest.raises(pkg.ConfigurationError):
        pkg.get_backend("blas")
    with pytest.raises(pkg.ConfigurationError):
        pkg.BuildConfig(thread_count=0)
    lay = pkg.AtomBlockLayout((4,))
    coeffs = pkg.StackedCoefficients(pkg.ComplexDense.zeros(4, 6), pkg.ComplexDense.zeros(4, 6),
                                     lay, np.ones(4))
    z = [pkg.ComplexDense.zeros(4, 4)]
    tm = pkg.TMatrixSet(z, z, z, [1], [1])
    with pytest.raises(pkg.ConfigurationError):
        pkg.build_all(coeffs, tm, pkg.BuildConfig(backup=False))


def test_ctypes_structs_match_the_c_header(tmp_path):
    """Every argument block the Python side passes through the C ABI has the header's field
    names, offsets and size (gcc compiles the header and prints offsetof / sizeof)."""
    import ctypes
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    from paper_1602_06589_b200 import _native

    structs = {"hsdla_ab_args": _native.AbArgs, "hsdla_reduced_args": _native.ReducedArgs,
               "hsdla_build_args": _native.BuildArgs, "hsdla_build_result": _native.BuildResult,
               "hsdla_c64": _native.C64}
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "hsdla_b200.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(out[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(out[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_tmatrixset_validate_structure():
    """builder.py:123-138: Hermitian residual and the dense-block + diagonal-tail pattern."""
    import numpy as np

    import paper_1602_06589_b200 as pkg

    rng = np.random.default_rng(3)
    m, d = 9, 4  # l_sph 2, l_nonsph 1
    t = np.zeros((m, m), dtype=np.complex128)
    x = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    t[:d, :d] = x + x.conj().T
    t[np.diag_indices(m)] += 3.0
    cd = pkg.ComplexDense.from_array
    ok = pkg.TMatrixSet([cd(t)], [cd(t)], [cd(t)], [2], [1])
    ok.validate_structure()
    bad = t.copy()
    bad[6, 2] = 0.1
    bad[2, 6] = 0.1
    with pytest.raises(pkg.ContractViolationError):
        pkg.TMatrixSet([cd(bad)], [cd(t)], [cd(t)], [2], [1]).validate_structure()
    nh = t.copy()
    nh[1, 0] += 0.5
    with pytest.raises(pkg.ContractViolationError):
        pkg.TMatrixSet([cd(t)], [cd(t)], [cd(nh)], [2], [1]).validate_structure()
