"""D2H rate of the pinned 144 MB H / S copies alone and while the GPU is loaded (the e2e path's
copies run under the contractions): idle, under an FP64 DGEMM loop (tensor pipe, little HBM
traffic), under an HBM copy loop, and under the C2 device-resident pipeline itself.  Also one
144 MB copy split into 1 / 2 / 4 pieces and pinned buffers from cudaHostAlloc vs
cudaHostRegister'd pageable memory.  Tells whether the e2e's ~51 GB/s under load (vs ~56 idle)
is the kernels' doing or the link's."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

n = 2999
nb = n * n * 16
dev = torch.empty((n, n), dtype=torch.complex128, device="cuda")
dev.normal_()
host = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
cs = torch.cuda.Stream()
ls = torch.cuda.Stream()


def d2h_rate(reps=8, pieces=1, dst=host):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        with torch.cuda.stream(cs):
            e0.record(cs)
            step = (n + pieces - 1) // pieces
            for p in range(0, n, step):
                dst[p:p + step].copy_(dev[p:p + step], non_blocking=True)
            e1.record(cs)
        cs.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts)[1:-1]
    ms = sum(ts) / len(ts)
    return nb / (ms / 1e3) / 1e9, ms


def under(load_fn, label, **kw):
    # start the load, let it ramp, measure copies while it runs, then drain
    torch.cuda.synchronize()
    with torch.cuda.stream(ls):
        for _ in range(kw.pop("depth", 40)):
            load_fn()
    time.sleep(0.02)
    r, ms = d2h_rate(**kw)
    busy = not ls.query()
    ls.synchronize()
    print(f"{label:<44s} {r:6.1f} GB/s  {ms:.3f} ms per 144 MB  (load still running at end: {busy})",
          flush=True)


r, ms = d2h_rate()
print(f"{'idle':<44s} {r:6.1f} GB/s  {ms:.3f} ms per 144 MB", flush=True)
for p in (2, 4, 16):
    r, ms = d2h_rate(pieces=p)
    print(f"{'idle, ' + str(p) + ' pieces':<44s} {r:6.1f} GB/s  {ms:.3f} ms", flush=True)

a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
under(lambda: torch.mm(a, b, out=c), "under DGEMM 8192^3 loop (DMMA)", depth=6)
x = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
under(lambda: y.copy_(x), "under 2 GB HBM copy loop", depth=60)
del a, b, c, x, y

from paper_1602_06589_b200 import configs  # noqa: E402
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats  # noqa: E402

inst = configs.make_instance("C2")
dspec = DeviceSpec(inst.spec)
tp = pack_tmats(inst.tmats)
pipe = HSPipeline(inst.spec.n_basis, dspec.heights)
for _ in range(3):
    pipe.run(dspec, tp)
torch.cuda.synchronize()
tickets = []


def c2_load():
    # device-resident builds on the pipeline's own stream (the library's compute stream)
    tickets.append(pipe.run_async(dspec, tp))
    if len(tickets) > 1:
        pipe.finish(tickets.pop(0))


c2_load()
ts = []
for _ in range(8):
    c2_load()  # the next k-point is queued before each copy: the copy runs under its contraction
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs)
        host.copy_(dev, non_blocking=True)
        e1.record(cs)
    cs.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = sorted(ts)[1:-1]
ms = sum(ts) / len(ts)
print(f"{'under the C2 pipeline (merged S+H contractions)':<44s} {nb / (ms / 1e3) / 1e9:6.1f} GB/s  {ms:.3f} ms",
      flush=True)
while tickets:
    pipe.finish(tickets.pop(0))
torch.cuda.synchronize()
r, ms = d2h_rate()
print(f"{'idle again':<44s} {r:6.1f} GB/s  {ms:.3f} ms", flush=True)
