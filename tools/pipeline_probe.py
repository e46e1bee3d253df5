"""Host-side timing of the pipelined k-point batch (build_hs_many) on one config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1602_06589_b200 import configs, BuildConfig
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats, _pinned_pair

inst = configs.make_instance(sys.argv[1] if len(sys.argv) > 1 else "C2")
spec = inst.spec
n = spec.n_basis
tp = pack_tmats(inst.tmats)
d0 = DeviceSpec(spec)
pipe = HSPipeline(n, d0.heights)
bufs = [_pinned_pair(n), _pinned_pair(n)]
for _ in range(3):
    pipe.run(d0, tp)
torch.cuda.synchronize()
K = 12
tt = {"spec": 0.0, "enqueue": 0.0, "finish": 0.0}
t_start = time.perf_counter()
pending = None
for i in range(K):
    t0 = time.perf_counter(); d = DeviceSpec(spec); t1 = time.perf_counter()
    tk = pipe.run_async(d, tp, host_out=bufs[i % 2]); t2 = time.perf_counter()
    tt["spec"] += t1 - t0; tt["enqueue"] += t2 - t1
    if pending is not None:
        t3 = time.perf_counter(); r = pipe.finish(pending); tt["finish"] += time.perf_counter() - t3
    pending = tk
r = pipe.finish(pending)
torch.cuda.synchronize()
total = time.perf_counter() - t_start
print(f"per k-point: {1e3*total/K:.3f} ms; host spec {1e3*tt['spec']/K:.3f}, enqueue {1e3*tt['enqueue']/K:.3f}, "
      f"finish-wait {1e3*tt['finish']/K:.3f}; last ms_total {r['ms_total']:.3f} kernel_ms {r['kernel_ms']}")
# without copies, for reference
t_start = time.perf_counter(); pending = None
for i in range(K):
    d = DeviceSpec(spec)
    tk = pipe.run_async(d, tp)
    if pending is not None:
        pipe.finish(pending)
    pending = tk
pipe.finish(pending); torch.cuda.synchronize()
print(f"no-copy pipelined per k-point: {1e3*(time.perf_counter()-t_start)/K:.3f} ms")
