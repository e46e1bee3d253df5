"""Which H form the reference-generated bundles take (GPU probe, not a test): joint factor,
structure split, HPD mask per T set."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
from paper_1602_06589_b200 import bundle, device
from paper_1602_06589_b200.pipeline import build_device, pack_tmats, padded_ld

for name in ("phys", "rand"):
    spec, co, tm = bundle.load_bundle(os.path.join("tests", "golden", "bundles", name))
    lay, n = co.layout, co.n_basis
    r = lay.total_rows
    ld = padded_ld(r)
    a_d = device.upload_window(co.A_star.array, ld)
    b_d = device.upload_window(co.B_star.array, ld)
    udot = torch.zeros(ld, dtype=torch.float64, device="cuda")
    udot[:r] = torch.from_numpy(np.ascontiguousarray(co.udot_norms)).cuda()
    h_d, s_d = device.empty_matrix(n, n, n), device.empty_matrix(n, n, n)
    tp = pack_tmats(tm)
    res, _ = build_device(n_basis=n, heights=lay.block_heights, row_offset=lay.offsets[:-1],
                          tpack=tp, A=a_d, B=b_d, Bs=None, udot=udot, ld=ld,
                          force_general_path=False, H=h_d, S=s_d, ldh=n)
    print(name, "t_dim", list(tp.t_dim), "t_dense", list(tp.t_dense), "joint", res["joint_t"],
          "split", res["joint_split"], "hpd", res["hpd_mask"])
