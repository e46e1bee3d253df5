"""T preparation timing (tprep_kernel, tjoint_kernel) on first builds of C2 and C4 (run under
ncu's launch list, or read the per-phase split): one fresh T pack per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1602_06589_b200 import configs  # noqa: E402
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats  # noqa: E402

for name in sys.argv[1:] or ["C2", "C4"]:
    inst = configs.make_instance(name)
    spec = inst.spec
    if name == "C4":  # the T preparation does not depend on N_G: a short G-set keeps this quick
        from bench import cpu_sample

        spec = cpu_sample(inst, 2000)
    ds = DeviceSpec(spec)
    pipe = HSPipeline(spec.n_basis, ds.heights)
    res = pipe.run(ds, pack_tmats(inst.tmats))
    torch.cuda.synchronize()
    print(name, "joint", res["joint_t"], "ms", res["ms"], flush=True)
