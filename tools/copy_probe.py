"""D2H bandwidth alone vs concurrent with the contraction kernels."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1602_06589_b200 import configs
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats

inst = configs.make_instance("C2")
spec = inst.spec
n = spec.n_basis
tp = pack_tmats(inst.tmats); d0 = DeviceSpec(spec); pipe = HSPipeline(n, d0.heights)
pipe.run(d0, tp)
src = torch.empty(n * n, dtype=torch.complex128, device="cuda")
dst = torch.empty(n * n, dtype=torch.complex128, pin_memory=True)
cs = torch.cuda.Stream()
def copy_time():
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs); dst.copy_(src, non_blocking=True); e1.record(cs)
    return e0, e1
torch.cuda.synchronize()
e0, e1 = copy_time(); torch.cuda.synchronize()
print(f"alone: {e0.elapsed_time(e1):.3f} ms for {n*n*16/1e6:.0f} MB")
# concurrent: enqueue compute on the current stream, then the copy on cs
for trial in range(3):
    torch.cuda.synchronize()
    pipe_ticket = pipe.run_async(d0, tp)
    e0, e1 = copy_time()
    r = pipe.finish(pipe_ticket); torch.cuda.synchronize()
    print(f"concurrent: copy {e0.elapsed_time(e1):.3f} ms; build ms_total {r['ms_total']:.3f}")
# copy via the pipeline's own path (host_out) vs none
ho = (torch.empty((n, n), dtype=torch.complex128, pin_memory=True), torch.empty((n, n), dtype=torch.complex128, pin_memory=True))
for trial in range(3):
    r = pipe.run(d0, tp, host_out=ho); print("run+host_out ms_total", round(r['ms_total'], 3), r['kernel_ms'])
    r = pipe.run(d0, tp); print("run          ms_total", round(r['ms_total'], 3))
