"""HSM1 files, bundles and the build flow (reference `matrix.py:242-276`, `cli.py:203-328`).

Golden bundles and their H/S come from the real reference CLI (tests/golden/make_bundles.py).
CPU tests: the host HSM1 reader/writer contract (reference test_matrix_core.py:155-222
restated), bundle loading and re-writing byte for byte, CLI exit codes that need no GPU.
GPU tests: build_bundle vs the reference's H.hsm1 / S.hsm1 / report.json, and the HBM
streaming reader/writer vs the host format.
"""
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, rand_complex, rel_fro

from paper_1602_06589_b200 import ComplexDense, ConfigurationError, ContractViolationError
from paper_1602_06589_b200.bundle import build_bundle, load_bundle, write_bundle
from paper_1602_06589_b200.hsm1 import (HSM1_MAGIC, read_hsm1, read_hsm1_device, write_hsm1,
                                        write_hsm1_device)

BUNDLES = os.path.join(GOLDEN, "bundles")


def _bundle(name):
    return os.path.join(BUNDLES, name)


# -- host HSM1 contract -----------------------------------------------------------------

def test_hsm1_round_trip_compacts(tmp_path):
    rng = np.random.default_rng(3)
    m = ComplexDense.from_array(rand_complex(rng, 6, 4))
    write_hsm1(tmp_path / "m.hsm1", m)
    back = read_hsm1(tmp_path / "m.hsm1")
    assert back.shape == (6, 4)
    np.testing.assert_array_equal(back.array, m.array)
    assert back.leading_dimension == 6


def test_hsm1_bytes(tmp_path):
    m = ComplexDense.from_array(np.array([[1 + 2j, 3 + 4j], [5 + 6j, 7 + 8j]]))
    write_hsm1(tmp_path / "m.hsm1", m)
    raw = (tmp_path / "m.hsm1").read_bytes()
    assert raw[:8] == HSM1_MAGIC == b"HSDLAM1\x00"
    assert int.from_bytes(raw[8:16], "little") == 2 and int.from_bytes(raw[16:24], "little") == 2
    np.testing.assert_array_equal(np.frombuffer(raw[24:], "<f8"), [1, 2, 5, 6, 3, 4, 7, 8])


def test_hsm1_window_compacted(tmp_path):
    rng = np.random.default_rng(4)
    big = ComplexDense.zeros(9, 3, capacity_rows=9)
    big.array[:] = rand_complex(rng, 9, 3)
    view = big.block(3, 4)
    write_hsm1(tmp_path / "v.hsm1", view)
    np.testing.assert_array_equal(read_hsm1(tmp_path / "v.hsm1").array, view.array)


def test_hsm1_errors(tmp_path):
    (tmp_path / "bad.hsm1").write_bytes(b"NOTHSM1\x00" + bytes(32))
    with pytest.raises(ValueError, match="magic"):
        read_hsm1(tmp_path / "bad.hsm1")
    (tmp_path / "short.hsm1").write_bytes(HSM1_MAGIC + bytes(4))
    with pytest.raises(ValueError, match="truncated"):
        read_hsm1(tmp_path / "short.hsm1")
    write_hsm1(tmp_path / "t.hsm1", ComplexDense.zeros(3, 3))
    data = (tmp_path / "t.hsm1").read_bytes()
    (tmp_path / "t.hsm1").write_bytes(data[:-8])
    with pytest.raises(ValueError, match="payload"):
        read_hsm1(tmp_path / "t.hsm1")
    m = ComplexDense.zeros(2, 2)
    m.array[1, 0] = np.nan
    with pytest.raises(ContractViolationError):
        write_hsm1(tmp_path / "x.hsm1", m)


def test_hsm1_empty(tmp_path):
    write_hsm1(tmp_path / "e.hsm1", ComplexDense.zeros(0, 5))
    back = read_hsm1(tmp_path / "e.hsm1")
    assert back.shape == (0, 5)


# -- bundles on the host ------------------------------------------------------------------

@pytest.mark.parametrize("name", ["phys", "rand"])
def test_load_and_rewrite_bundle_bytewise(tmp_path, name):
    """Reading a reference bundle and writing it back reproduces every file byte for byte."""
    spec, coeffs, tmats = load_bundle(_bundle(name))
    manifest = json.loads(open(os.path.join(_bundle(name), "manifest.json")).read())
    assert coeffs.n_basis == manifest["n_basis"]
    assert coeffs.A_star.leading_dimension == coeffs.layout.capacity_rows
    assert (spec is None) == (name == "rand")
    out = write_bundle(tmp_path / name, coeffs, tmats, spec, seed=manifest["seed"],
                       params=manifest["params"])
    assert out["files"] == manifest["files"]
    assert json.loads((tmp_path / name / "manifest.json").read_text()) == manifest


def test_cli_exit_codes_without_gpu(tmp_path):
    from paper_1602_06589_b200.__main__ import main

    assert main(["build", str(tmp_path / "missing")]) == 2            # IO error
    assert main(["build", _bundle("rand"), "--no-backup",
                 "--out", str(tmp_path / "o")]) == 1                   # needs system.json
    assert main(["build", _bundle("rand"), "--threads", "0"]) == 1
    assert main(["frobnicate"]) == 1
    with pytest.raises(ConfigurationError, match="system.json"):
        build_bundle(_bundle("rand"), tmp_path / "o2", backup=False)


# -- GPU: the build flow against the reference's own outputs -------------------------------

def _report_core(doc):
    return {k: v for k, v in doc.items() if not k.startswith("time_") and k != "peak_observed_bytes"}


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["phys", "rand"])
def test_build_bundle_matches_reference(cuda, tmp_path, name):
    outdir, report = build_bundle(_bundle(name), tmp_path / "out")
    ref = _bundle(name + "_out")
    for mat in ("H", "S"):
        got = read_hsm1(outdir / f"{mat}.hsm1").array
        want = read_hsm1(os.path.join(ref, f"{mat}.hsm1")).array
        assert got.shape == want.shape
        assert rel_fro(got, want) <= 1e-12, (mat, rel_fro(got, want))
        np.testing.assert_array_equal(got, got.conj().T)           # exact Hermitian output
    mine = json.loads((outdir / "report.json").read_text())
    theirs = json.loads(open(os.path.join(ref, "report.json")).read())
    assert _report_core(mine) == _report_core(theirs)
    assert report.ledger.total == theirs["flops_total"]


@pytest.mark.gpu
def test_build_bundle_backup_modes_bitwise(cuda, tmp_path):
    a, _ = build_bundle(_bundle("phys"), tmp_path / "a", backup=True)
    b, _ = build_bundle(_bundle("phys"), tmp_path / "b", backup=False)
    for mat in ("H.hsm1", "S.hsm1"):
        assert (a / mat).read_bytes() == (b / mat).read_bytes()


@pytest.mark.gpu
def test_cli_build(cuda, tmp_path):
    from paper_1602_06589_b200.__main__ import main

    assert main(["build", _bundle("phys"), "--out", str(tmp_path / "o")]) == 0
    assert (tmp_path / "o" / "H.hsm1").is_file() and (tmp_path / "o" / "report.json").is_file()


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,ld,panel", [(37, 53, 48, 16 * 37 * 5), (64, 7, 64, 1 << 20),
                                                (1, 300, 16, 160), (5, 1, 5, 1 << 20)])
def test_hsm1_device_stream_matches_host_format(cuda, tmp_path, rows, cols, ld, panel):
    """HBM -> file streaming (several panels, ld > rows windows) writes exactly the host
    writer's bytes, and file -> HBM reads them back with zero padding rows."""
    rng = np.random.default_rng(rows * 1000 + cols)
    host = rand_complex(rng, rows, cols)
    dev = cuda.zeros((cols, ld), dtype=cuda.complex128, device="cuda")
    dev[:, :rows] = cuda.from_numpy(np.ascontiguousarray(host.T)).cuda()
    n = write_hsm1_device(tmp_path / "d.hsm1", dev, rows, cols, panel_bytes=panel)
    write_hsm1(tmp_path / "h.hsm1", ComplexDense.from_array(host))
    assert (tmp_path / "d.hsm1").read_bytes() == (tmp_path / "h.hsm1").read_bytes()
    assert n == 24 + 16 * rows * cols
    back, r, c = read_hsm1_device(tmp_path / "h.hsm1", ld + 3, panel_bytes=panel)
    assert (r, c) == (rows, cols) and tuple(back.shape) == (cols, ld + 3)
    b = back.cpu().numpy()
    np.testing.assert_array_equal(b[:, :rows].T, host)
    assert not b[:, rows:].any()


@pytest.mark.gpu
def test_hsm1_device_guards(cuda, tmp_path):
    dev = cuda.zeros((4, 4), dtype=cuda.complex128, device="cuda")
    dev[2, 3] = complex(float("inf"), 0.0)
    with pytest.raises(ContractViolationError, match="non-finite"):
        write_hsm1_device(tmp_path / "x.hsm1", dev, 4, 4)
    assert not (tmp_path / "x.hsm1").exists()
    # the non-finite element outside the written window is not looked at
    write_hsm1_device(tmp_path / "ok.hsm1", dev, 3, 4)
    write_hsm1_device(tmp_path / "e.hsm1", dev, 0, 4)
    assert read_hsm1(tmp_path / "e.hsm1").shape == (0, 4)
    (tmp_path / "bad.hsm1").write_bytes(b"XXXXXXXX" + bytes(16))
    with pytest.raises(ValueError, match="magic"):
        read_hsm1_device(tmp_path / "bad.hsm1")
    shutil.copy(os.path.join(_bundle("rand"), "A.hsm1"), tmp_path / "a.hsm1")
    data = (tmp_path / "a.hsm1").read_bytes()
    (tmp_path / "a.hsm1").write_bytes(data[:-16])
    with pytest.raises(ValueError, match="payload"):
        read_hsm1_device(tmp_path / "a.hsm1")
