"""Measured parity against the REAL reference's own H / S (tests/golden/big_*.npz, made by
tests/golden/make_golden_big.py) for both B200 entry points, as numbers rather than pass/fail:

    python tools/parity_table.py > profiles/r02c_parity_vs_reference.json

Per config: relative Frobenius error of the stored panel columns, the random columns and the
projections H V / S V, and the largest entrywise deviation relative to the largest entry."""
import json
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")

import paper_1602_06589_b200 as pkg  # noqa: E402
from paper_1602_06589_b200 import configs  # noqa: E402
from paper_1602_06589_b200.builder import release_cached_workspaces  # noqa: E402
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def stats(g, key, panel, cols, proj):
    ref_p, ref_c = g[f"{key}_panel"], g[f"{key}_cols"]
    return {"panel_rel_fro": rel(panel, ref_p), "cols_rel_fro": rel(cols, ref_c),
            "proj_rel_fro": rel(proj, g[f"{key}V"]),
            "max_entry_dev_over_max_entry": float(max(np.abs(panel - ref_p).max(),
                                                      np.abs(cols - ref_c).max())
                                                  / np.abs(ref_p).max())}


def main():
    out = {}
    for name in ("C2", "C3", "C4", "C5", "C2NS", "C2IND"):
        g = np.load(os.path.join(GOLDEN, f"big_{name}.npz"))
        inst = configs.make_instance(name)
        spec, n = inst.spec, inst.spec.n_basis
        dspec = DeviceSpec(spec)
        pipe = HSPipeline(n, dspec.heights)
        pipe.run(dspec, pack_tmats(inst.tmats))
        h_t, s_t = pipe.result_views()
        vt = torch.from_numpy(g["V"]).cuda()

        def cols(t, idx):
            return t[torch.from_numpy(np.asarray(idx)).cuda()].cpu().numpy().T

        rec = {"n_basis": n, "rows": int(dspec.rows), "pipeline": {}, "dropin": {}}
        for key, t in (("H", h_t), ("S", s_t)):
            rec["pipeline"][key] = stats(g, key, cols(t, g["panel"]), cols(t, g["cols"]),
                                         (t.transpose(0, 1) @ vt).cpu().numpy())
        del pipe, h_t, s_t
        coeffs = pkg.compute_AB(spec)
        h, s, _ = pkg.build_all(coeffs, inst.tmats, pkg.BuildConfig())
        for key, m in (("H", h.array), ("S", s.array)):
            rec["dropin"][key] = stats(g, key, m[:, g["panel"]], m[:, g["cols"]], m @ g["V"])
        out[name] = rec
        del coeffs, h, s
        release_cached_workspaces()
        torch.cuda.empty_cache()
    print(json.dumps({"what": "B200 H / S vs the unmodified reference's own output (goldens), "
                              "bar 1e-12", "configs": out}, indent=1))


if __name__ == "__main__":
    main()
