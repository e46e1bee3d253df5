"""Import shim (test infrastructure): the reference's own test suite run against the B200 package.

With `tests/ref_shim` first on sys.path, `import hsdla` gives the reference's public names
bound to `paper_1602_06589_b200` (compute on the GPU through libhsdla_b200.so), so the
reference's pkg/tests/{test_kernels,test_builder,test_matrix_core}.py run unchanged against
it (SURVEY.md §4 reuse plan).  The few names the tests need that are not part of the hot path
come from the reference itself, installed under baseline/_ref (the reference arm's install):
its naive numba oracle (`naive_H`, `naive_S`, `compare_matrices`: the tests' ground truth) and
its input synthesis (`synth_T`, `synth_coefficients`, outputs re-wrapped as this package's
types sharing the same buffers).
"""
import importlib.util
import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if _REPO not in sys.path:
    sys.path.insert(0, _REPO)

import paper_1602_06589_b200 as _b200  # noqa: E402
from paper_1602_06589_b200 import *  # noqa: E402,F401,F403
from paper_1602_06589_b200 import (ComplexDense, StackedCoefficients,  # noqa: E402
                                   TMatrixSet)

REF_ROOT = os.environ.get("HSDLA_REF_ROOT") or os.path.join(_REPO, "baseline", "_ref", "hsdla")


def _load_reference():
    """The reference package under the private name `_hsdla_reference` (relative imports
    resolve inside it), so it does not collide with this shim's `hsdla`."""
    name = "_hsdla_reference"
    if name in sys.modules:
        return sys.modules[name]
    init = os.path.join(REF_ROOT, "__init__.py")
    if not os.path.exists(init):
        raise ImportError(f"reference package not installed at {REF_ROOT} (bench arm install)")
    spec = importlib.util.spec_from_file_location(name, init, submodule_search_locations=[REF_ROOT])
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


_ref = _load_reference()


def _wrap(m):
    """A reference ComplexDense as this package's type over the same allocation."""
    return ComplexDense(m._base, m._row0, m.rows)


def synth_T(*args, **kwargs):
    t = _ref.synth_T(*args, **kwargs)
    return TMatrixSet([_wrap(x) for x in t.t_aa], [_wrap(x) for x in t.t_ab],
                      [_wrap(x) for x in t.t_bb], list(t.l_sph), list(t.l_nonsph))


def synth_coefficients(seed, layout, *args, **kwargs):
    c = _ref.synth_coefficients(seed, layout, *args, **kwargs)
    return StackedCoefficients(_wrap(c.A_star), _wrap(c.B_star), layout, c.udot_norms)


def naive_S(coeffs):
    return _wrap(_ref.naive_S(coeffs))


def naive_H(coeffs, tmats):
    return _wrap(_ref.naive_H(coeffs, tmats))


compare_matrices = _ref.compare_matrices
naive_flop_count = _ref.naive_flop_count
__version__ = _b200.__version__
