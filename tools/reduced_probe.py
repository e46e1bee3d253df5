"""Reduced A-side overlap vs the stacked contraction A*^H A* (GPU probe, not a test).

Times hsdla_reduced_s_aa (inputs resident in HBM) and the DMMA herk of A* for the same
spec; prints both, the agreement, and the reduced kernel's arithmetic rate.
"""
import ctypes, json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1602_06589_b200 as p
from paper_1602_06589_b200 import _native, configs, device
from paper_1602_06589_b200.reduced import ReducedPlan, reduced_overlap_inputs


def ev_time(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for cfg in sys.argv[1:] or ["C2", "C3"]:
    spec = configs.make_instance(cfg).spec
    n = spec.n_basis
    inp = reduced_overlap_inputs(spec)
    out = torch.empty((n, n), dtype=torch.complex128, device="cuda")
    plan = ReducedPlan(inp)
    ms_red = ev_time(lambda: plan.run(out))
    coeffs = p.compute_AB(spec)
    r = coeffs.layout.total_rows
    a = device.upload_window(coeffs.A_star.array)
    c = torch.zeros((n, n), dtype=torch.complex128, device="cuda")
    lib = _native.load()
    herk = lambda: _native.check(lib.hsdla_herk_lower(device.ctx(), n, r, device.ptr(a), a.shape[1],
                                                      device.ptr(c), n), "herk")
    c.zero_(); herk(); torch.cuda.synchronize()
    low = torch.tril(c.T)  # (row, col) lower of the stacked result
    red = out.T
    err = (torch.linalg.norm(torch.tril(red) - low) / torch.linalg.norm(low)).item()
    ms_herk = ev_time(herk)
    l1 = int(spec.l_sph.max()) + 1
    print(json.dumps({"config": cfg, "n_basis": n, "atoms": spec.n_atoms, "l_max": l1 - 1,
                      "reduced_ms": round(ms_red, 4), "stacked_herk_ms": round(ms_herk, 4),
                      "speedup": round(ms_herk / ms_red, 2), "rel_err_lower": err,
                      "types": plan.n_types,
                      "reduced_gflops_est": round(n * (n + 1) / 2 * (8 * spec.n_atoms + 8 * l1 * plan.n_types) / ms_red / 1e9, 1)}),
          flush=True)
