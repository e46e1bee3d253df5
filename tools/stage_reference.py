"""Install the reference package for the reference arm and stage its own test files (build
container only; needs /root/reference).  Outputs are git-ignored and travel to the GPU box with
the repo snapshot:

* baseline/_ref/hsdla        — `pip install --no-index --no-build-isolation --no-deps --target
                               baseline/_ref` of a /tmp copy of /root/reference/pkg (the tree is
                               read-only; dependency resolution is skipped: numpy, scipy, numba
                               and threadpoolctl are already in the image);
* baseline/_ref/hsdla_tests  — the reference's pkg/tests/*.py, unmodified, run by
                               tests/test_ref_suite.py against this package (import shim) and
                               with the B200 backend inside the reference (pytest plugin).
"""
import os
import shutil
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference"
DEST = os.path.join(REPO, "baseline", "_ref")


def main() -> int:
    if not os.path.isdir(REF):
        print("stage_reference: /root/reference absent (GPU box): nothing to stage")
        return 0
    if not os.path.exists(os.path.join(DEST, "hsdla", "__init__.py")):
        with tempfile.TemporaryDirectory() as tmp:
            src = os.path.join(tmp, "pkg")
            shutil.copytree(os.path.join(REF, "pkg"), src)
            subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
                            "--no-deps", "--find-links", "/opt/wheelhouse", "--target", DEST, src],
                           check=True, capture_output=True)
    tests = os.path.join(DEST, "hsdla_tests")
    os.makedirs(tests, exist_ok=True)
    for f in sorted(os.listdir(os.path.join(REF, "pkg", "tests"))):
        if f.endswith(".py"):
            shutil.copy2(os.path.join(REF, "pkg", "tests", f), os.path.join(tests, f))
    with open(os.path.join(tests, "pytest.ini"), "w") as fh:
        fh.write("[pytest]\naddopts = -p no:cacheprovider\n")
    print(f"stage_reference: {DEST} ready")
    return 0


if __name__ == "__main__":
    sys.exit(main())
