"""Time the drop-in reference API on the GPU: compute_AB(spec) then build_all(coeffs, ...), and
the fused single call pipeline.build_hs, with the native build timeline (HSDLA_TIMELINE) and a
host-side profile of one build_all call."""
import cProfile
import os
import pstats
import sys
import time

os.environ.setdefault("HSDLA_TIMELINE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1602_06589_b200 as p  # noqa: E402
from paper_1602_06589_b200 import configs  # noqa: E402
from paper_1602_06589_b200.pipeline import build_hs  # noqa: E402

inst = configs.make_instance(sys.argv[1] if len(sys.argv) > 1 else "C2")
for rep in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    co = p.compute_AB(inst.spec)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    h, s, r = p.build_all(co, inst.tmats, p.BuildConfig())
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"drop-in: compute_AB {1e3*(t1-t0):.2f} ms  build_all {1e3*(t2-t1):.2f} ms  total {1e3*(t2-t0):.2f} ms", flush=True)
    del h, s, co
out = None
for rep in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h, s, r = build_hs(inst.spec, inst.tmats, host_out=out)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    out = (torch.from_numpy(h.base.T), torch.from_numpy(s.base.T))
    print(f"build_hs single call {1e3*(t1-t0):.2f} ms", flush=True)
co = p.compute_AB(inst.spec)
pr = cProfile.Profile()
pr.enable()
h, s, r = p.build_all(co, inst.tmats, p.BuildConfig())
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
