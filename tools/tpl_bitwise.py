"""Dump one C2 device-pipeline build (H, S) for a bitwise comparison between library variants
(GPU probe: run twice under different HSDLA_* switches, then compare the .npy files)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1602_06589_b200 import configs  # noqa: E402
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats  # noqa: E402

name, out = sys.argv[1], sys.argv[2]
inst = configs.make_instance(name)
d = DeviceSpec(inst.spec)
pipe = HSPipeline(inst.spec.n_basis, d.heights)
r = pipe.run(d, pack_tmats(inst.tmats))
h, s = (x.cpu().numpy() for x in pipe.result_views())
np.savez(out, h=h, s=s, types=r["template_types"])
