"""Golden H / S data at BASELINE sizes made by running the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden_big.py

Imports `hsdla` from /root/reference/pkg/src (read-only; not available on the GPU box) and
runs its own `compute_AB` (flapw.py:201-233) + `build_all` (builder.py:403-474, optimized
backend on every host thread) on the seeded BASELINE systems of paper_1602_06589_b200.configs:

* big_C2.npz — C2 (N_G 2999, R 1296)
* big_C3.npz — C3 (N_G 7994, R 5184)
* big_C4.npz — C4 (N_G 12986, R 13068, three atom types; ~25 min and ~25 GB of host memory here)
* big_C5.npz — C5's first k-point (N_G ~5000, R 2592)
* big_C2NS.npz, big_C2IND.npz — the C2-sized non-BASELINE systems with structured T (l_nonsph 6:
  the T-structure split) and indefinite T (no T_AA is HPD: the shifted joint form on the GPU,
  the general ZHEMM/ZGEMM path in the reference)

Each file holds, for H and S: full columns of the middle 64-column panel (all 64 at C2 / C3, the
first 32 / 16 of it at C5 / C4 to keep the fixtures small; they cross every tile row of that
panel), random full columns, H V / S V for seeded random V, the diagonals,
the Frobenius norms, plus the ledger, the HPD mask and digests of the inputs (the GPU tests
rebuild the inputs from configs.py and refuse to compare if they drifted).  The full
matrices (144 MB / 1 GB each) are not stored.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import hsdla  # noqa: E402  (the reference)

from paper_1602_06589_b200 import configs  # noqa: E402

sys.path.insert(0, HERE)
from digest import input_digest  # noqa: E402

COLS = {"C2": 16, "C3": 16, "C4": 8, "C5": 12, "C2NS": 8, "C2IND": 8}
PANEL_COLS = {"C2": 64, "C3": 64, "C4": 16, "C5": 32, "C2NS": 16, "C2IND": 16}


def main(names):
    for name in names:
        inst = configs.make_instance(name)
        spec = hsdla.SystemSpec.from_json_dict(inst.spec.to_json_dict())
        cd = hsdla.ComplexDense.from_array
        tm = inst.tmats
        rtm = hsdla.TMatrixSet(t_aa=[cd(t.array) for t in tm.t_aa], t_ab=[cd(t.array) for t in tm.t_ab],
                               t_bb=[cd(t.array) for t in tm.t_bb], l_sph=list(tm.l_sph),
                               l_nonsph=list(tm.l_nonsph))
        t0 = time.time()
        coeffs = hsdla.compute_AB(spec)
        t1 = time.time()
        h, s, rep = hsdla.build_all(coeffs, rtm, hsdla.BuildConfig(backend="optimized",
                                                                    thread_count=os.cpu_count()))
        t2 = time.time()
        H, S = h.array, s.array
        n = H.shape[0]
        nb = (n + 63) // 64
        j0 = 64 * (nb // 2)
        panel = np.arange(j0, min(n, j0 + PANEL_COLS[name]))
        rng = np.random.default_rng(2024)
        cols = np.sort(rng.choice(np.setdiff1d(np.arange(n), np.arange(j0, min(n, j0 + 64))),
                                  size=COLS[name], replace=False))
        v = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
        out = {
            "digest": np.array(input_digest(inst)), "n": n, "panel": panel, "cols": cols,
            "H_panel": H[:, panel], "S_panel": S[:, panel], "H_cols": H[:, cols], "S_cols": S[:, cols],
            "V": v, "HV": H @ v, "SV": S @ v, "H_diag": np.diag(H).copy(), "S_diag": np.diag(S).copy(),
            "H_fro": np.linalg.norm(H), "S_fro": np.linalg.norm(S),
            "ledger_total": rep.ledger.total, "hpd_mask": np.array(rep.hpd_mask, dtype=bool),
            "seconds": np.array([t1 - t0, t2 - t1]),
        }
        np.savez(os.path.join(HERE, f"big_{name}.npz"), **out)
        print(f"{name}: N={n} compute_AB {t1 - t0:.1f} s build_all {t2 - t1:.1f} s "
              f"({os.cpu_count()} threads)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3"])
