"""Run one C1/C2 build_all and save H, S (GPU probe, not a test): compare HSDLA_CMUL modes.

    HSDLA_CMUL=3 python tools/cmul_compare.py C2 out3.npz; HSDLA_CMUL=4 ... out4.npz
    python tools/cmul_compare.py --diff out3.npz out4.npz   (on any host; + oracle errors)
"""
import sys
import numpy as np
sys.path.insert(0, ".")

if sys.argv[1] == "--diff":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in ("h", "s"):
        d = np.linalg.norm(a[k] - b[k]) / np.linalg.norm(b[k])
        print(k, "rel_fro(3 vs 4) =", f"{d:.3e}", "bitwise equal:", np.array_equal(a[k], b[k]))
    if "ho" in a:
        for k in ("h", "s"):
            for nm, x in (("3", a), ("4", b)):
                print(k, nm, "vs oracle", f"{np.linalg.norm(x[k] - a[k + 'o']) / np.linalg.norm(a[k + 'o']):.3e}")
    sys.exit(0)

import paper_1602_06589_b200 as pkg
from paper_1602_06589_b200 import configs
cfg, out = sys.argv[1], sys.argv[2]
inst = configs.make_instance(cfg)
coeffs = pkg.compute_AB(inst.spec)
h, s, rep = pkg.build_all(coeffs, inst.tmats, pkg.BuildConfig())
extra = {}
if len(sys.argv) > 3:
    from oracle import build as ob, flapw as of
    a, b, norms, offs = of.compute_ab(inst.spec)
    tm = inst.tmats
    ho, so, _, _ = ob.build_all(a, b, norms, list(np.diff(offs)), [t.array for t in tm.t_aa],
                                [t.array for t in tm.t_ab], [t.array for t in tm.t_bb])
    extra = {"ho": ho, "so": so}
np.savez(out, h=h.array, s=s.array, **extra)
print("saved", out)
