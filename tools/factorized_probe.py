"""Per-type factorised build vs the stacked pipeline, end to end (spec + T -> host H, S)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1602_06589_b200 import configs
from paper_1602_06589_b200.factorized import atom_types, build_hs_factorized, build_hs_factorized_device
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats
from paper_1602_06589_b200.pipeline import build_hs


def wall(fn, reps):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e3, out


for cfg in sys.argv[1:] or ["C2", "C3"]:
    inst = configs.make_instance(cfg)
    reps = 3 if cfg in ("C1", "C2", "C5") else 1
    tf, (hf, sf, _) = wall(lambda: build_hs_factorized(inst.spec, inst.tmats), reps)
    ts, (hs, ss, _) = wall(lambda: build_hs(inst.spec, inst.tmats), reps)
    td, _ = wall(lambda: build_hs_factorized_device(inst.spec, inst.tmats), reps)
    pipe = HSPipeline(inst.spec.n_basis, DeviceSpec(inst.spec).heights)
    dsp, tp = DeviceSpec(inst.spec), pack_tmats(inst.tmats)
    tsd, _ = wall(lambda: pipe.run(dsp, tp), reps)
    err = max(np.linalg.norm(hf.array - hs.array) / np.linalg.norm(hs.array),
              np.linalg.norm(sf.array - ss.array) / np.linalg.norm(ss.array))
    print(json.dumps({"config": cfg, "n_basis": inst.spec.n_basis, "atoms": inst.spec.n_atoms,
                      "types": len(atom_types(inst.spec, inst.tmats)),
                      "factorized_ms": round(tf, 2), "stacked_ms": round(ts, 2),
                      "factorized_device_ms": round(td, 2), "stacked_device_ms": round(tsd, 2),
                      "speedup": round(ts / tf, 2), "rel_diff": err}), flush=True)
