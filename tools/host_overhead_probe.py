"""Host-side cost of one synchronous call (GPU probe, not a test): wall time of build_hs vs its
device timeline, and a cProfile of the steady-state calls (where the host time goes)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1602_06589_b200 import BuildConfig, configs  # noqa: E402
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, build_hs, pack_tmats  # noqa: E402

inst = configs.make_instance(sys.argv[1] if len(sys.argv) > 1 else "C2")
spec = inst.spec
pipe = HSPipeline(spec.n_basis, DeviceSpec(spec).heights)
host_out = None
for i in range(4):
    h, s, r = build_hs(spec, inst.tmats, BuildConfig(), pipeline=pipe, host_out=host_out)
    host_out = (torch.from_numpy(h.base.T), torch.from_numpy(s.base.T))
walls = []
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h, s, r = build_hs(spec, inst.tmats, BuildConfig(), pipeline=pipe, host_out=host_out)
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
print("wall ms", [round(w, 3) for w in walls])
for name, fn in (("DeviceSpec", lambda: DeviceSpec(spec)), ("pack_tmats", lambda: pack_tmats(inst.tmats))):
    t0 = time.perf_counter()
    for _ in range(20):
        fn()
    print(name, "ms", round((time.perf_counter() - t0) * 1e3 / 20, 3))
pr = cProfile.Profile()
pr.enable()
for i in range(5):
    h, s, r = build_hs(spec, inst.tmats, BuildConfig(), pipeline=pipe, host_out=host_out)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
