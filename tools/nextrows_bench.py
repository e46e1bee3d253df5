"""Measurements of the SURVEY §8(f) rows beside their CPU counterparts (GPU probe, not a test):

  * row 1 `verify`: the GPU build plus the independent GPU evaluation of the defining sums
    (verify.verify_metrics) at C2, beside the oracle port's build_all (the CPU path) on the
    same inputs;
  * row 2 HSM1 output: H and S of a C2 build streamed from HBM into HSM1 files
    (write_hsm1_device) and read back into HBM (read_hsm1_device), beside the reference
    format routine on host arrays (write_hsm1 on the same matrices);
  * row 4 Gaunt-sum T assembly (assemble_T on the GPU) for a C2NS-like type (l_sph 8,
    l_nonsph 6, 16 atoms) beside the oracle's numpy restatement;
  * row 3 (Legendre-reduced S_AA, per-type factorisation) is measured by
    tools/reduced_probe.py / tools/factorized_probe.py (profiles/r01_*_probe.jsonl).

Prints one JSON object.  Oracle imports are CPU baselines only (bench.py's rule)."""
import json
import os
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_06589_b200 as pkg  # noqa: E402
from paper_1602_06589_b200 import configs, hsm1, verify  # noqa: E402
from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats  # noqa: E402


def best(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


out = {"box_threads": os.cpu_count()}

# ---- row 1: verify at C2 ---------------------------------------------------------------------
inst = configs.make_instance("C2")
coeffs = pkg.compute_AB(inst.spec)
verify.verify_metrics(inst.spec, coeffs, inst.tmats)  # warm-up (T preparation, workspaces)
metrics = {}


def run_verify():
    metrics.update(verify.verify_metrics(inst.spec, coeffs, inst.tmats))


v_ms = best(run_verify, 2)
from oracle import flapw as of  # noqa: E402  (CPU baseline)
from oracle import build as ob  # noqa: E402

a, b, norms, offs = of.compute_ab(inst.spec)
tm = inst.tmats
t0 = time.perf_counter()
ob.build_all(a, b, norms, list(np.diff(offs)), [t.array for t in tm.t_aa], [t.array for t in tm.t_ab],
             [t.array for t in tm.t_bb])
cpu_build_ms = (time.perf_counter() - t0) * 1e3
out["verify_C2"] = {"gpu_ms": round(v_ms, 2), "rel_err_H": metrics["rel_err_H"],
                    "rel_err_S": metrics["rel_err_S"], "s_hpd": metrics["s_hpd"],
                    "cpu_oracle_build_all_ms": round(cpu_build_ms, 1),
                    "what": "GPU build_all + independent GPU evaluation of the defining sums + "
                            "Hermitian residuals + S Cholesky (verify_metrics); CPU: the oracle's "
                            "build_all alone on the same inputs (scipy OpenBLAS)"}

# ---- row 2: HSM1 streaming -------------------------------------------------------------------
dspec = DeviceSpec(inst.spec)
pipe = HSPipeline(inst.spec.n_basis, dspec.heights)
pipe.run(dspec, pack_tmats(inst.tmats))
h_dev, s_dev = pipe.result_views()  # (column, row) storage, n x n
n = inst.spec.n_basis
with tempfile.TemporaryDirectory() as d:
    ph, ps = os.path.join(d, "H.hsm1"), os.path.join(d, "S.hsm1")

    def w_dev():
        hsm1.write_hsm1_device(ph, h_dev, n, n)
        hsm1.write_hsm1_device(ps, s_dev, n, n)

    wd_ms = best(w_dev)

    def r_dev():
        hsm1.read_hsm1_device(ph)
        hsm1.read_hsm1_device(ps)

    rd_ms = best(r_dev)
    h_host = pkg.ComplexDense(h_dev[:n, :n].cpu().numpy().T)
    s_host = pkg.ComplexDense(s_dev[:n, :n].cpu().numpy().T)

    def w_host():
        hsm1.write_hsm1(ph, h_host)
        hsm1.write_hsm1(ps, s_host)

    wh_ms = best(w_host)
    nbytes = 2 * (16 * n * n + 16)
out["hsm1_C2"] = {"bytes": nbytes, "write_from_hbm_ms": round(wd_ms, 1),
                  "read_into_hbm_ms": round(rd_ms, 1), "write_host_arrays_ms": round(wh_ms, 1),
                  "write_from_hbm_gbs": round(nbytes / wd_ms / 1e6, 2),
                  "read_into_hbm_gbs": round(nbytes / rd_ms / 1e6, 2),
                  "what": "H and S of one C2 build (2 x 144 MB) to HSM1 files in a temporary "
                          "directory of the box and back; host: the reference's format routine "
                          "on host copies of the same matrices"}

# ---- row 4: Gaunt-sum T assembly ---------------------------------------------------------------
ns = configs.make_instance("C2NS")
spec = ns.spec
ints = [pkg.synth_radial_integrals(100 + a, int(spec.l_nonsph[a])) for a in range(spec.n_atoms)]
pkg.assemble_T(spec, ints)  # warm-up (Gaunt tensor)
ta_ms = best(lambda: pkg.assemble_T(spec, ints))
from oracle import assemble as oa  # noqa: E402  (CPU baseline)

energies = [np.asarray(spec.radial[a].energy) for a in range(spec.n_atoms)]
udn = [np.asarray(spec.radial[a].udot_norm) for a in range(spec.n_atoms)]
t0 = time.perf_counter()
oa.assemble_T([int(x) for x in spec.l_sph], [int(x) for x in spec.l_nonsph], energies, udn,
              [(r.c_uu, r.c_ud, r.c_dd) for r in ints])
cpu_ta_ms = (time.perf_counter() - t0) * 1e3
out["assemble_T_C2NS"] = {"atoms": spec.n_atoms, "l_sph": int(spec.l_sph[0]),
                          "l_nonsph": int(spec.l_nonsph[0]), "gpu_ms": round(ta_ms, 2),
                          "cpu_oracle_ms": round(cpu_ta_ms, 1),
                          "what": "per-atom T_AA, T_AB, T_BB from Gaunt sums (hsdla_gaunt_sum) "
                                  "incl. the integrals' pairing checks and host copies; CPU: "
                                  "oracle/assemble.py (numpy einsum, Gaunt tensor per atom)"}
print(json.dumps(out, indent=1))
