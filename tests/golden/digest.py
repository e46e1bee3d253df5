"""Digest of the seeded inputs a golden fixture was made from (shared by the generator and the
tests, so a change of configs.py is caught instead of compared against stale data)."""
import hashlib

import numpy as np


def input_digest(inst) -> str:
    """sha256 over the spec arrays, radial data and T blocks of a configs.Instance."""
    h = hashlib.sha256()
    sp = inst.spec
    for arr in (sp.k_vectors, sp.positions, sp.rotations, sp.mt_radius):
        h.update(np.ascontiguousarray(arr, dtype=np.float64).tobytes())
    for rad in sp.radial:
        for f in ("u", "u_prime", "udot", "udot_prime", "udot_norm"):
            h.update(np.ascontiguousarray(getattr(rad, f), dtype=np.float64).tobytes())
    for fam in (inst.tmats.t_aa, inst.tmats.t_ab, inst.tmats.t_bb):
        for t in fam:
            h.update(np.ascontiguousarray(t.array).tobytes())
    return h.hexdigest()
