import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from conftest import rel_fro
from paper_1602_06589_b200 import configs
from paper_1602_06589_b200.pipeline import build_hs, build_hs_many, HSPipeline, DeviceSpec
inst = configs.make_instance("C1")
tm = inst.tmats
allspecs = [configs.kpoint_variant(inst, r) for r in range(4)]
ref = {id(s): build_hs(s, tm)[0].array.copy() for s in allspecs}
print("sizes", [s.n_basis for s in allspecs])
for order in ([0, 1, 2], [2, 1, 0], [1, 0, 2], [0, 0, 0], [0, 2], [2, 0], [1, 2], [0, 1, 2, 3]):
    specs = [allspecs[i] for i in order]
    n_cap = max(s.n_basis for s in specs)
    pipe = HSPipeline(n_cap, DeviceSpec(specs[0]).heights)
    got = {}
    build_hs_many(specs, tm, pipeline=pipe, on_result=lambda i, h, s, r: got.__setitem__(i, h.array.copy()))
    torch.cuda.synchronize()
    errs = [rel_fro(got[i], ref[id(s)]) for i, s in enumerate(specs)]
    n = specs[-1].n_basis
    dev = pipe.H[:n, :n].cpu().numpy().T
    print(order, [s.n_basis for s in specs], ["%.1e" % e for e in errs], "device-last-vs-ref %.1e" % rel_fro(dev, ref[id(specs[-1])]))
