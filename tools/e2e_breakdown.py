"""Time the pieces of the e2e path (build_hs) on C2: host prep, native call, copies."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1602_06589_b200 import configs
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats

inst = configs.make_instance(sys.argv[1] if len(sys.argv) > 1 else "C2")
spec = inst.spec
n = spec.n_basis
dspec = DeviceSpec(spec)
pipe = HSPipeline(n, dspec.heights)
tp = pack_tmats(inst.tmats)
host = (torch.empty((n, n), dtype=torch.complex128, pin_memory=True),
        torch.empty((n, n), dtype=torch.complex128, pin_memory=True))
for _ in range(3):
    pipe.run(dspec, tp, host_out=host)
torch.cuda.synchronize()
for rep in range(5):
    t0 = time.perf_counter(); d = DeviceSpec(spec); torch.cuda.synchronize(); t1 = time.perf_counter()
    tpk = pack_tmats(inst.tmats); torch.cuda.synchronize(); t2 = time.perf_counter()
    r = pipe.run(d, tpk, host_out=host); t3 = time.perf_counter()
    r2 = pipe.run(d, tpk); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"DeviceSpec {1e3*(t1-t0):.3f} ms  pack_tmats {1e3*(t2-t1):.3f} ms  run+copy {1e3*(t3-t2):.3f} ms "
          f"(events {r['ms_total']:.3f})  run-no-copy {1e3*(t4-t3):.3f} ms (events {r2['ms_total']:.3f})")
x = torch.empty(n * n * 2, dtype=torch.complex128, device="cuda")
h = torch.empty(n * n * 2, dtype=torch.complex128, pin_memory=True)
torch.cuda.synchronize(); t0 = time.perf_counter(); h.copy_(x); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"plain D2H {x.numel()*16/1e6:.0f} MB: {1e3*(t1-t0):.3f} ms = {x.numel()*16/(t1-t0)/1e9:.1f} GB/s")
