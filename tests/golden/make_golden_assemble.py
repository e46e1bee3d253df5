"""Golden fixtures for the input-side Gaunt machinery, made by running the REAL reference
(build container only; /root/reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden_assemble.py

* assemble_t.npz — gaunt_tensor(3, 2) and gaunt_tensor(2, 2) (special.py:227-244), a few
  gaunt() values incl. refine=2 (special.py:207-224), synth_radial_integrals for three atoms
  (flapw.py:289-307) and assemble_T's per-atom T_AA / T_AB / T_BB (flapw.py:310-363) on a
  synth_system spec with mixed l_sph / l_nonsph.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import hsdla  # noqa: E402  (the reference)
from hsdla import special  # noqa: E402


def main():
    out = {}
    out["g32"] = special.gaunt_tensor(3, 2)
    out["g22"] = special.gaunt_tensor(2, 2)
    triples = [((1, 0), (1, 0), (0, 0)), ((2, 1), (1, 1), (1, 0)), ((3, -2), (2, -1), (1, -1)),
               ((4, 3), (3, 2), (2, 1))]
    out["gaunt_args"] = np.array([[a[0], a[1], b[0], b[1], c[0], c[1]] for a, b, c in triples])
    out["gaunt_vals"] = np.array([special.gaunt(a, b, c) for a, b, c in triples])
    out["gaunt_vals_refine2"] = np.array([special.gaunt(a, b, c, refine=2) for a, b, c in triples])
    spec = hsdla.synth_system(31, 3, [4, 3, 5], [2, 3, 1], basis_factor=50.0)
    ris = [hsdla.synth_radial_integrals(40 + a, int(spec.l_nonsph[a])) for a in range(3)]
    tm = hsdla.assemble_T(spec, ris)
    out["l_sph"] = np.asarray(spec.l_sph)
    out["l_nonsph"] = np.asarray(spec.l_nonsph)
    for a in range(3):
        out[f"energy{a}"] = spec.radial[a].energy
        out[f"udot_norm{a}"] = spec.radial[a].udot_norm
        for f in ("c_uu", "c_dd", "c_ud", "c_du"):
            out[f"{f}{a}"] = getattr(ris[a], f)
        out[f"t_aa{a}"] = tm.t_aa[a].array
        out[f"t_ab{a}"] = tm.t_ab[a].array
        out[f"t_bb{a}"] = tm.t_bb[a].array
    np.savez_compressed(os.path.join(HERE, "assemble_t.npz"), **out)
    print("wrote assemble_t.npz")


if __name__ == "__main__":
    main()
