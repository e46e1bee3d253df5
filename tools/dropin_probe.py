"""Time the drop-in reference API on the GPU: compute_AB(spec) then build_all(coeffs, ...)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1602_06589_b200 as p
from paper_1602_06589_b200 import configs
inst = configs.make_instance(sys.argv[1] if len(sys.argv) > 1 else "C2")
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    co = p.compute_AB(inst.spec)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    h, s, r = p.build_all(co, inst.tmats, p.BuildConfig())
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"compute_AB {1e3*(t1-t0):.2f} ms  build_all {1e3*(t2-t1):.2f} ms  total {1e3*(t2-t0):.2f} ms")
