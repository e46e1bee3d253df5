"""Indefinite T (GPU probe): BASELINE distributions with the diagonal shift -2, and T_BB scaled by
||udot|| on both sides as the physics scales it (<udot|H|udot> ~ E ||udot||^2), so the common
shift sigma ~ |lambda_min| passes the amplification guard.  Device time per k-point and H
agreement: shifted joint form vs the reference forms."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1602_06589_b200 import ComplexDense, TMatrixSet, configs
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
inst = configs.make_instance(cfg, hpd_shift=-2.0)
spec, tm = inst.spec, inst.tmats
# rescale T_BB per T object by the (shared) ||udot|| rows of its atoms
scaled = {}
t_bb = []
for a in range(spec.n_atoms):
    key = id(tm.t_bb[a])
    if key not in scaled:
        l = int(spec.l_sph[a])
        u = np.repeat(np.asarray(spec.radial[a].udot_norm[:l + 1]), 2 * np.arange(l + 1) + 1)
        scaled[key] = ComplexDense.from_array(u[:, None] * tm.t_bb[a].array * u[None, :])
    t_bb.append(scaled[key])
tm = TMatrixSet(tm.t_aa, tm.t_ab, t_bb, tm.l_sph, tm.l_nonsph)
d = DeviceSpec(spec)
tp = pack_tmats(tm)
hs = []
for ref_form in (False, True):
    pipe = HSPipeline(spec.n_basis, d.heights, h_reference_form=ref_form)
    for _ in range(3):
        r = pipe.run(d, tp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        r = pipe.run(d, tp)
    e1.record()
    torch.cuda.synchronize()
    hs.append(pipe.result_views()[0].clone())
    print(f"{cfg} indefinite T, {'reference forms' if ref_form else 'shifted joint  '}: "
          f"{e0.elapsed_time(e1) / 10:.3f} ms  joint {all(r['joint_t'])} sigma {r['joint_shift']:.3g} "
          f"hpd {sum(r['hpd_mask'])}/{len(r['hpd_mask'])}")
diff = torch.linalg.norm(hs[0] - hs[1]) / torch.linalg.norm(hs[1])
print(f"{cfg}: rel_fro(H shifted joint, H reference forms) = {diff.item():.2e}")
