"""Single-call build timelines with host destinations (GPU probe, not a test): compute events
and copy-completion events per build (HSDLA_TIMELINE=1 prints them from the library)."""
import os
import sys
os.environ["HSDLA_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time
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
for _ in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe.run(dspec, tp, host_out=host)
    print(f"wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
