"""Steady-state k-point interval of build_hs_many (host-observed completions) vs the device
step time; shows whether e2e loses time per k-point or only in pipeline fill/drain."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1602_06589_b200 import BuildConfig, configs
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, build_hs_many

inst = configs.make_instance(sys.argv[1] if len(sys.argv) > 1 else "C2")
spec = inst.spec
pipe = HSPipeline(spec.n_basis, DeviceSpec(spec).heights)
bufs = {}
build_hs_many([spec] * 3, inst.tmats, BuildConfig(), pipeline=pipe, host_buffers=bufs)
for rep in range(2):
    stamps = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rr = build_hs_many([spec] * 30, inst.tmats, BuildConfig(), pipeline=pipe, host_buffers=bufs,
                       on_result=lambda i, h, s, r: stamps.append(time.perf_counter()))
    t1 = time.perf_counter()
    iv = [1e3 * (b - a) for a, b in zip(stamps, stamps[1:])]
    print(f"total {1e3*(t1-t0)/30:.3f} ms/kpt; first completion {1e3*(stamps[0]-t0):.2f} ms; "
          f"steady interval median {statistics.median(iv):.3f} ms (min {min(iv):.3f}, max {max(iv):.3f}); "
          f"device ms_total median {statistics.median(r['ms_total'] for r in rr):.3f}")
ks = {}
for r in rr[2:]:
    for k, v in r["kernel_ms"].items():
        ks.setdefault(k, []).append(v)
print("kernel_ms during the batch:", {k: round(statistics.median(v), 4) for k, v in ks.items()})
ticket_ms = []
for _ in range(10):
    r = pipe.run(DeviceSpec(spec), rr and __import__("paper_1602_06589_b200.pipeline", fromlist=["x"]).pack_tmats(inst.tmats))
    ticket_ms.append(r["kernel_ms"])
print("kernel_ms without host copies:", {k: round(statistics.median(x[k] for x in ticket_ms), 4) for k in ticket_ms[0]})
