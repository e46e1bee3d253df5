"""`python -m paper_1602_06589_b200 verify` (the reference CLI's verify, cli.py:331-409) on
bundles written by the reference CLI itself, against the verdicts and verify.json the reference
produced for them (tests/golden/make_bundles.py): exit 0 on the physics, random and small
(2R >= N_G: S Cholesky) bundles; exit 4 with the same failing metrics on the bundle with a
de-Hermitised T_BB; exit 1 above the N_G guard without --force."""
import json
import os
import subprocess
import sys

import pytest

from conftest import GOLDEN, REPO

pytestmark = pytest.mark.gpu
B = os.path.join(GOLDEN, "bundles")


def _verify(tmp_path, name, *extra):
    out = tmp_path / f"{name}_v"
    r = subprocess.run([sys.executable, "-m", "paper_1602_06589_b200", "verify",
                        os.path.join(B, name), "--out", str(out), *extra],
                       cwd=REPO, capture_output=True, text=True, timeout=600)
    got = json.loads((out / "verify.json").read_text()) if (out / "verify.json").exists() else None
    return r.returncode, r.stdout, got, r.stderr


@pytest.mark.parametrize("name", ["phys", "rand", "small"])
def test_verify_passes_like_reference(cuda, tmp_path, name):
    rc, stdout, got, stderr = _verify(tmp_path, name)
    ref = json.loads(open(os.path.join(B, f"{name}_verify", "verify.json")).read())
    assert rc == 0, stdout + stderr
    assert "verification passed" in stdout
    assert got["s_hpd"] == ref["s_hpd"]
    for k in ("rel_err_H", "rel_err_S", "herm_residual_H_oracle", "herm_residual_S_oracle"):
        assert got[k] <= 1e-13, (k, got[k])
    # the build report inside verify.json: the reference's ledger and HPD accounting
    for k in ("flops_total", "hpd_atom_count", "non_hpd_atom_count", "predicted_bytes"):
        assert got["report"][k] == ref["report"][k], k


def test_verify_flags_de_hermitised_t_bb(cuda, tmp_path):
    rc, stdout, got, stderr = _verify(tmp_path, "phys_fault")
    ref = json.loads(open(os.path.join(B, "phys_fault_verify", "verify.json")).read())
    ref_rc = int(open(os.path.join(B, "phys_fault_verify", "exit_code.txt")).read())
    assert rc == ref_rc == 4, stdout
    keys = ("rel_err_H", "rel_err_S", "herm_residual_H_oracle", "herm_residual_S_oracle")
    fails = {k for k in keys if got[k] > 1e-11}
    ref_fails = {k for k in keys if ref[k] > 1e-11}
    assert fails == ref_fails == {"rel_err_H", "herm_residual_H_oracle"}
    # the independent evaluation reproduces the reference oracle's numbers
    for k in ("rel_err_H", "herm_residual_H_oracle"):
        assert abs(got[k] / ref[k] - 1) <= 1e-10, (k, got[k], ref[k])
    assert "verification FAILED: rel_err_H, herm_residual_H_oracle" in stdout


def test_verify_size_guard(cuda, tmp_path, monkeypatch):
    import paper_1602_06589_b200.verify as v

    monkeypatch.setattr(v, "ORACLE_SIZE_GUARD", 8)
    from paper_1602_06589_b200 import ConfigurationError

    with pytest.raises(ConfigurationError):
        v.cmd_verify(os.path.join(B, "phys"), echo=lambda *_: None)
    assert v.cmd_verify(os.path.join(B, "phys"), force=True, echo=lambda *_: None) == 0
