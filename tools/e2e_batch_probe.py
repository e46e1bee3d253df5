"""The e2e k-point batch (pipeline.build_hs_many, C2) against this box's pure D2H rate: is the
batch at the copy floor (288 MB of H and S per k-point), or does the copy engine idle between
k-points?  With HSDLA_TIMELINE=1 the library prints each build's S / H copy completion times
(ms since the context epoch) on stderr; this script prints wall ms per k-point and the floor."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1602_06589_b200 import BuildConfig, configs
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, build_hs_many

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 30
inst = configs.make_instance(cfg)
spec = inst.spec
n = spec.n_basis
d = torch.empty((n, n), dtype=torch.complex128, device="cuda")
h = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
torch.cuda.synchronize()
ts = []
for _ in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms_copy = sorted(ts)[len(ts) // 2]
rate = n * n * 16 / (ms_copy / 1e3) / 1e9
print(f"pure D2H: {rate:.1f} GB/s; floor per k-point (H + S) {2 * ms_copy:.3f} ms", flush=True)
del d, h
specs = [spec] * count
pipe = HSPipeline(n, DeviceSpec(spec).heights)
bufs = {}
build_hs_many(specs[:3], inst.tmats, BuildConfig(), pipeline=pipe, host_buffers=bufs)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    build_hs_many(specs, inst.tmats, BuildConfig(), pipeline=pipe, host_buffers=bufs)
    torch.cuda.synchronize()
    print(f"batch of {count}: {(time.perf_counter() - t0) * 1e3 / count:.3f} ms per k-point",
          flush=True)
