"""The reference's OWN test files (pkg/tests/test_kernels.py, test_builder.py,
test_matrix_core.py, staged unmodified under baseline/_ref/hsdla_tests by tools/stage_reference.py)
run two ways (SURVEY.md §4 reuse plan):

* shim    — `import hsdla` resolves to tests/ref_shim: the reference's names bound to this
            package (every build and operator on the GPU); the conftest's backend names
            "reference" / "optimized" both select the B200 backend;
* backend — the unmodified reference package (baseline/_ref) with the B200 operators registered
            into its `_BACKENDS` under both names (tests/ref_plugin, `integration.py`): the
            reference's own builder drives the sm_100a kernels.

Each run is a pytest subprocess; the test asserts exit 0 and the pass count."""
import os
import re
import subprocess
import sys

import pytest

from conftest import REPO

REF_TESTS = os.path.join(REPO, "baseline", "_ref", "hsdla_tests")
REF_PKG = os.path.join(REPO, "baseline", "_ref")


def _run(tmp_path, mode, files, extra=()):
    if not os.path.exists(os.path.join(REF_TESTS, "test_kernels.py")) or \
            not os.path.exists(os.path.join(REF_PKG, "hsdla", "__init__.py")):
        pytest.skip("reference package / tests not staged (tools/stage_reference.py)")
    env = dict(os.environ, NUMBA_CACHE_DIR=str(tmp_path / "numba"), PYTHONDONTWRITEBYTECODE="1")
    if mode == "shim":
        env["PYTHONPATH"] = os.path.join(REPO, "tests", "ref_shim")
        plugin = []
    else:
        env["PYTHONPATH"] = os.pathsep.join([REF_PKG, os.path.join(REPO, "tests", "ref_plugin")])
        plugin = ["-p", "b200_backend_plugin"]
    cmd = [sys.executable, "-m", "pytest", "-q", "--rootdir", REF_TESTS, *plugin, *extra,
           *[os.path.join(REF_TESTS, f) for f in files]]
    out = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True,
                         timeout=1800)
    tail = (out.stdout + out.stderr)[-3000:]
    m = re.search(r"(\d+) passed", out.stdout)
    return out.returncode, int(m.group(1)) if m else 0, tail


def test_reference_matrix_core_suite_host_parts(tmp_path):
    """CPU: the storage contract (ComplexDense windows, layout, ledger, HSM1 byte layout) of the
    reference's test_matrix_core.py against this package; the device helpers (scale_rows,
    mirror) are the GPU run's."""
    rc, passed, tail = _run(tmp_path, "shim", ["test_matrix_core.py"],
                            ["-k", "not scale_rows and not mirror"])
    assert rc == 0, tail
    assert passed >= 15, tail


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["shim", "backend"])
def test_reference_suite_on_b200(cuda, tmp_path, mode):
    rc, passed, tail = _run(tmp_path, mode, ["test_kernels.py", "test_builder.py",
                                             "test_matrix_core.py"])
    assert rc == 0, tail
    assert passed >= 120, tail  # 66 kernel + 43 builder + 22 matrix-core cases in the reference
