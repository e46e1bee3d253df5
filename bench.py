"""Benchmark of the muffin-tin H/S setup (FLAPW, HSDLA) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one k-point of the BASELINE configuration through the hot path
(A/B generation + Cholesky/T application + the S and H triangular DMMA contractions
with the fused Hermitian mirror), inputs (SystemSpec, T blocks) resident in HBM.
The metric is BASELINE.json's: H+S setup time per k-point and FP64 TFLOP/s over the
reference's nominal FLOP ledger (`builder.py:336-370`), as a fraction of the measured
FP64 DMMA peak.  Multi-GPU: one process per GPU (torchrun), each rank builds its own
k-point (k-point parallelism, weak scaling, no collective in the data path); the
time is the max over ranks.  `--impl reference` times the unmodified reference package
(baseline/_ref, installed by tools/stage_reference.py: its own compute_AB + build_all,
"optimized" backend on every host thread; `cpu_baseline.kind` "reference") on the host
cores, rank 0 only, with the numpy oracle port beside it (`oracle_port`); where the package
is not installed the port is the arm (`kind` "port").  Prints one JSON line.
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = ("H+S setup time per k-point & FP64 TFLOP/s (fraction of B200 FP64 peak), "
          "1/2/4/8 GPU")
UNIT = "TFLOP/s"
FP64_PEAK_TFLOPS = 37.2  # measured DMMA ceiling, profiles/r01_fp64_peaks.json (= 148*128*1.965 GHz)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="C2",
                   choices=["C1", "C2", "C3", "C4", "C5", "C2NS", "C2IND"],
                   help="BASELINE.json configs C1-C5; not BASELINE configs: C2NS = C2 with "
                        "l_nonsph = 6 < l_sph = 8 (structured T), C2IND = C2 with indefinite T")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--mode", default="kpoints", choices=["kpoints", "panels"],
                   help="kpoints: one k-point per GPU per step (weak scaling, default); "
                        "panels: ONE k-point split over all GPUs by column panels, "
                        "gathered to rank 0 (strong scaling)")
    p.add_argument("--panel-transport", default="nccl", choices=["nccl", "p2p"],
                   help="panel gather: nccl = batched send/recv + mirror on rank 0 (default); "
                        "p2p = tiles and their mirror stored into rank 0's symmetric-memory "
                        "H/S by the contraction epilogue (after a self-test; nccl if it fails)")
    p.add_argument("--no-extras", action="store_true",
                   help="skip the BASELINE scaling configs (C5 k-point batch, C3 panels) "
                        "reported as extra keys of the line")
    p.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                   help=argparse.SUPPRESS)  # gloo: multi-rank flow check, ranks may share a GPU
    p.add_argument("--dry-run", action="store_true",
                   help="launcher check without a GPU: spawn the ranks (gloo), deal the "
                        "work, print one JSON line; no compute")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ CPU oracle leg

def cpu_oracle_step(spec, tmats):
    """One k-point through the oracle port; returns (seconds, ledger FLOPs)."""
    from oracle import build as ob
    from oracle import flapw as of

    t0 = time.perf_counter()
    a, b, norms, offs = of.compute_ab(spec)
    t1 = time.perf_counter()
    _, _, led, _ = ob.build_all(a, b, norms, list(np.diff(offs)), [t.array for t in tmats.t_aa],
                                [t.array for t in tmats.t_ab], [t.array for t in tmats.t_bb])
    t2 = time.perf_counter()
    return t2 - t0, sum(led.values()), t1 - t0, t2 - t1


def reference_package():
    """The real reference (`hsdla`, unmodified) installed by tools/stage_reference.py under
    baseline/_ref (git-ignored; travels to the GPU box with the snapshot), or None."""
    global _REF_PKG
    if _REF_PKG is not False:
        return _REF_PKG
    _REF_PKG = None
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")
    if os.environ.get("HSDLA_BENCH_CPU_ARM") == "port":  # force the oracle port
        return None
    if os.path.exists(os.path.join(path, "hsdla", "__init__.py")):
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_hsdla_ref")
        sys.path.insert(0, path)
        try:
            import hsdla

            if os.path.abspath(hsdla.__file__).startswith(path):
                _REF_PKG = hsdla
        except Exception as exc:  # pragma: no cover
            print(f"bench: reference package not importable ({exc}); CPU arm uses the oracle port",
                  file=sys.stderr)
        finally:
            sys.path.remove(path)
    return _REF_PKG


_REF_PKG = False


def cpu_reference_step(spec, tmats):
    """One k-point through the unmodified reference's own entry points: compute_AB
    (flapw.py:201-233) + build_all (builder.py:403-474, its "optimized" backend on every host
    thread).  Same return as cpu_oracle_step."""
    ref = reference_package()
    rspec = ref.SystemSpec.from_json_dict(spec.to_json_dict())
    cd = ref.ComplexDense.from_array
    rtm = ref.TMatrixSet(t_aa=[cd(t.array) for t in tmats.t_aa],
                         t_ab=[cd(t.array) for t in tmats.t_ab],
                         t_bb=[cd(t.array) for t in tmats.t_bb], l_sph=list(tmats.l_sph),
                         l_nonsph=list(tmats.l_nonsph))
    cfg = ref.BuildConfig(backend="optimized", thread_count=affinity_threads())
    t0 = time.perf_counter()
    coeffs = ref.compute_AB(rspec)
    t1 = time.perf_counter()
    _, _, rep = ref.build_all(coeffs, rtm, cfg)
    t2 = time.perf_counter()
    return t2 - t0, rep.ledger.total, t1 - t0, t2 - t1


def cpu_step_fn():
    """(step function, kind, label): the real reference when it is installed, else the port."""
    if reference_package() is not None:
        return cpu_reference_step, "reference", "reference hsdla compute_AB + build_all"
    return cpu_oracle_step, "port", "oracle compute_AB + build_all"


def cpu_sample(inst, max_basis=3200):
    """Bounded CPU workload: the config's k-point, truncated to the first `max_basis`
    K-vectors when larger (C3/C4), so one sample takes seconds, not minutes."""
    from paper_1602_06589_b200 import SystemSpec

    spec = inst.spec
    if spec.n_basis > max_basis:
        spec = SystemSpec(positions=spec.positions, rotations=spec.rotations,
                          mt_radius=spec.mt_radius, l_sph=spec.l_sph, l_nonsph=spec.l_nonsph,
                          k_point=spec.k_point, k_vectors=spec.k_vectors[:max_basis],
                          omega=spec.omega, radial=spec.radial)
    return spec


def host_threads():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max(int(i.get("num_threads", 1)) for i in info) if info else os.cpu_count()
    except Exception:  # pragma: no cover
        return os.cpu_count()


def affinity_threads():
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
               else (os.cpu_count() or 1))


def use_all_host_threads():
    """The CPU arms use every host thread: torchrun exports OMP_NUM_THREADS=1 to each rank,
    which would otherwise cap the reference's OpenBLAS at one thread."""
    try:
        from threadpoolctl import threadpool_limits

        n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        return threadpool_limits(limits=max(1, n), user_api="blas")
    except Exception:  # pragma: no cover
        return None


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    _limits = use_all_host_threads()  # noqa: F841 (kept alive for the run)
    from paper_1602_06589_b200 import configs

    inst = configs.make_instance(args.config)

    def sample_spec(k):  # distinct seeded k-points of the config, bounded in N_G
        one = configs.Instance(inst.cfg, [configs.kpoint_variant(inst, k)], inst.tmats,
                               inst.min_abs_wronskian)
        return cpu_sample(one)

    step, kind, label = cpu_step_fn()
    for _ in range(max(0, min(args.warmup, 1))):
        step(sample_spec(0), inst.tmats)
    times, flops, nb = [], 0, set()
    t_start = time.perf_counter()
    for k in range(args.steps):
        spec = sample_spec(k)
        nb.add(spec.n_basis)
        dt, fl, _, _ = step(spec, inst.tmats)
        times.append(dt)
        flops += fl
        if time.perf_counter() - t_start > 150:  # keep the arm within a few minutes
            break
    total = sum(times)
    value = flops / total / 1e12
    port = None
    if kind == "reference":  # the numpy port of the same path beside it (one k-point, untimed warm-up)
        cpu_oracle_step(sample_spec(0), inst.tmats)
        pdt, pfl, _, _ = cpu_oracle_step(sample_spec(0), inst.tmats)
        port = {"ms_per_step": round(1e3 * pdt, 3), "value": round(pfl / pdt / 1e12, 4),
                "unit": UNIT, "what": "oracle port (vectorised compute_AB + the same scipy BLAS "
                                      "calls), one k-point"}
    trunc = max(nb) < inst.spec.n_basis
    sample = (f"{len(times)} distinct seeded k-point(s) of {args.config}" +
              (f" truncated to N_G={max(nb)}" if trunc else f" (N_G {min(nb)}-{max(nb)})") +
              f": {label} (scipy OpenBLAS)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": max(world, args.gpus), "steps": len(times), "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / len(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, inst),
                   "n_basis": max(nb), "rows": int(sum((l + 1) ** 2 for l in inst.spec.l_sph))},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": host_threads(),
                         "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if port is not None:
        line["oracle_port"] = port
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._thr = threading.Thread(target=self._loop, daemon=True)
            self._thr.start()
        except Exception as e:  # pragma: no cover
            self.error = str(e)
        return self

    def _loop(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:  # pragma: no cover
                pass
            time.sleep(0.005)

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr:
            self._thr.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ GPU arm

def fp64_ceilings(sm_mhz):
    """the DMMA peak at boost clock and at the clock measured during the run, and
    the measured cuBLAS ZGEMM ceiling on the S-contraction shape (profiles/r01_fp64_peaks.json)."""
    out = {"dmma_peak_boost_tflops": FP64_PEAK_TFLOPS}
    if sm_mhz:
        out["dmma_peak_at_measured_clock_tflops"] = round(148 * 128 * float(sm_mhz) * 1e6 / 1e12, 2)
    try:
        with open(os.path.join(REPO, "profiles", "r01_fp64_peaks.json")) as f:
            z = json.load(f)["cublas_zgemm_tflops"]
        out["cublas_zgemm_3000x3000x2592_tflops"] = z.get("3000x3000x2592")
    except (OSError, KeyError, ValueError):
        pass
    return out


def hbm_peak_gbs():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6550.0, "SURVEY.md 8d measured copy bandwidth"


_WRITE_CEILING = {}


def write_ceiling_gbs(nbytes):
    """Measured write-only HBM rate for a pass of `nbytes` (torch fill_ of that many bytes, best
    of 8, CUDA events): the ceiling a write-only kernel of that size can reach on this box.
    Short passes do not reach the copy-bandwidth peak (ramp-up and tail): C2's 124 MB fill
    runs at ~5.0 TB/s, a 1.3 GB one at ~7.2 TB/s (profiles/r02_expand_variants.json)."""
    if nbytes in _WRITE_CEILING:
        return _WRITE_CEILING[nbytes]
    import torch
    x = torch.empty(max(1, nbytes // 16), dtype=torch.complex128, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(8):
        e0.record()
        x.fill_(1.0)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del x
    _WRITE_CEILING[nbytes] = round(nbytes / (best / 1e3) / 1e9, 1)
    return _WRITE_CEILING[nbytes]


def ab_gen_line(ms, rows, n, template_types=0, expand_w_ms=None, templates_ms=None):
    """A/B generation against the HBM-write roofline.  Per-atom path: the
    generator writes A*, B* and ||udot|| B* (48 R N bytes).  Template path: the
    per-type templates (negligible bytes, latency-bound recurrences) and the expansion pass
    writing A* and ||udot|| B* (32 R N bytes) make up `ms`; the second expansion, W1 and W2
    of the joint H form (32 R N bytes), is reported as `expand_W` (the reference's Bytes_AB
    counts A*, B* = 32 R N)."""
    peak, src = hbm_peak_gbs()
    written = (32 if template_types else 48) * rows * n
    gbs = written / (ms / 1e3) / 1e9
    out = {"ms": round(ms, 4), "bytes_written": written, "bytes_ab_ref": 32 * rows * n,
           "achieved_gbs": round(gbs, 1), "peak_gbs": peak, "peak_source": src,
           "frac": round(gbs / peak, 4),
           "path": (f"per-type templates ({template_types} type(s)) + expansion" if template_types
                    else "per-atom generator")}
    if template_types and templates_ms is not None and ms > templates_ms > 0:
        # the HBM-bound part alone: the expansion writing A*, ||udot|| B* after the templates
        xm = ms - templates_ms
        xg = written / (xm / 1e3) / 1e9
        wc = write_ceiling_gbs(written)
        out["templates_ms"] = round(templates_ms, 4)
        out["expand_AB"] = {"ms": round(xm, 4), "bytes_written": written,
                            "achieved_gbs": round(xg, 1), "frac": round(xg / peak, 4),
                            "write_ceiling_gbs": wc, "frac_of_write_ceiling": round(xg / wc, 4)}
    if template_types and expand_w_ms:
        w = 32 * rows * n
        wg = w / (expand_w_ms / 1e3) / 1e9
        wc = write_ceiling_gbs(w)
        out["expand_W"] = {"ms": round(expand_w_ms, 4), "bytes_written": w,
                           "achieved_gbs": round(wg, 1), "frac": round(wg / peak, 4),
                           "write_ceiling_gbs": wc, "frac_of_write_ceiling": round(wg / wc, 4)}
    if template_types:
        out["write_ceiling_source"] = ("torch fill_ of the same byte count on this GPU, best of 8 "
                                       "(a write-only pass of that size cannot beat it)")
    return out


def executed_flops(fc, kc_ms, products, n, rows, hpd_rows, joint_rows, hpd_joint_rows=None):
    """What the DMMA pipe actually executes in the two contractions, next to the reference
    ledger `fc` (the algorithmic flops `achieved` is computed from; `hpd_rows`, `hpd_joint_rows`
    do not change the executed count).  Two restructurings make
    the executed work smaller than the ledger: the H contraction of a T set whose joint matrix
    [[T_AA, T_AB], [T_AB^H, T_BB]] is HPD is one rank-2m update per atom (8 flops x 2m x N^2
    complex MACs-equivalent, K = 2R) instead of ZHER2K + ZHERK (K = 3R); and the kernel issues
    `products` real DMMA products per complex MAC (2 flops each) instead of the ledger's 8
    flops.  The executed-flop rate is the tensor-pipe utilisation."""
    # rows of the reference forms: ZHER2K over all of them plus ZHERK (HPD) or ZGEMM (not HPD)
    # over each; the kernel evaluates the ZGEMM's A^H X into the lower triangle only, like the
    # ZHERK, so both execute 4 flops-equivalents per row and N^2 (the ledger counts 8 for ZGEMM)
    del hpd_rows, hpd_joint_rows
    h_ref = 12 * (rows - joint_rows) * n * n
    complex_equiv = 8 * rows * n * n + 8 * joint_rows * n * n + h_ref
    ex = complex_equiv * 2 * products / 8
    tf = ex / (kc_ms / 1e3) / 1e12
    return {"complex_mul": f"{products}-product", "h_joint_rows": int(joint_rows),
            "executed_flops_per_step": int(ex), "executed_tflops": round(tf, 3),
            "executed_frac": round(tf / FP64_PEAK_TFLOPS, 4),
            "note": "executed = the DMMA products the kernels issue (three-product multiply, joint "
                    "T factor for H): the tensor-pipe utilisation"}


def joint_rows_of(dspec, tpack, res, hpd_only=False):
    """Stacked rows whose T set took the joint factor (result "joint_t" per T set); with
    `hpd_only` only those of atoms whose T_AA is HPD."""
    jt = res.get("joint_t", [])
    mask = res.get("hpd_mask", [True] * len(dspec.heights))
    return int(sum(h for h, t, m in zip(dspec.heights, tpack.t_index, mask)
                   if t < len(jt) and jt[t] and (m or not hpd_only)))


def contract_flops(n, rows, hpd_rows):
    """F_contract of the two triangular contractions: 8RN^2 (S) +
    8RN^2 (ZHER2K) + 4 R_hpd N^2 + 8 R_nonhpd N^2 — the ledger's share of the DMMA kernels."""
    return 16 * rows * n * n + 4 * hpd_rows * n * n + 8 * (rows - hpd_rows) * n * n


def workload_name(config: str, inst) -> str:
    """The `config.workload` string, identical in both arms for one --config."""
    spec = inst.spec
    heights = sorted({int((l + 1) ** 2) for l in spec.l_sph})
    rows = int(sum((l + 1) ** 2 for l in spec.l_sph))
    tag = (f"{config} (BASELINE.json configs[{int(config[1]) - 1}])" if len(config) == 2
           else f"{config} (not a BASELINE config)")
    if len(inst.specs) > 1:
        ng = [x.n_basis for x in inst.specs]
        return (f"{tag}: {len(inst.specs)} k-points, N_G {min(ng)}-{max(ng)}, N_A={spec.n_atoms}, "
                f"N_L={'/'.join(map(str, heights))}, R={rows}, one k-point per step")
    return (f"{tag}: N_G={spec.n_basis}, N_A={spec.n_atoms}, N_L={'/'.join(map(str, heights))}, "
            f"R={rows}, one k-point per step")


def init_dist(world: int, local: int, backend: str = "nccl"):
    import torch
    import torch.distributed as dist

    if world > 1 and not dist.is_initialized():
        import datetime

        # a rank that fails must not leave the others waiting in a collective for the default
        # half hour: give up after five minutes
        tmo = datetime.timedelta(seconds=300)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=tmo)
        else:
            dist.init_process_group(backend, timeout=tmo)
    return dist


def max_over_ranks(vals, world, op="max"):
    """Reduce a list of floats over the ranks (device tensor, NCCL)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(v) for v in vals], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


def time_kpoints(pipe, dspecs, tpack, steps, world):
    """Time `steps` k-points back to back through the pipelined native path (step i+1 is
    enqueued before step i is collected) with CUDA events on the compute stream, barrier +
    synchronize on both sides.  Returns (ms on this rank, per-kernel ms lists, A/B ms list,
    last result)."""
    import torch
    import torch.distributed as dist

    kern = collections.defaultdict(list)
    ab_ms = []
    stream = torch.cuda.current_stream()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    prev = None
    res = None

    def collect(ticket):
        nonlocal res
        res = pipe.finish(ticket)
        for k, v in res["kernel_ms"].items():
            kern[k].append(v)
        ab_ms.append(res["ms"]["setup"])  # A/B generation (T preparation reused)
        kern["templates"].append(res.get("ms_templates", 0.0))

    for i in range(steps):
        ticket = pipe.run_async(dspecs[i % len(dspecs)], tpack)
        if prev is not None:
            collect(prev)
        prev = ticket
    e1.record(stream)
    collect(prev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return e0.elapsed_time(e1), kern, ab_ms, res


def contraction_roofline(fc, kern, products, n, rows, hpd_rows, joint_rows, traffic=None):
    """roofline object of the dominant kernel (the S + H triangular DMMA contractions).

    `achieved` counts the flops of the algorithm the kernel executes — the S and H
    contractions with the three-product complex multiply and, for joint T sets, H as one
    rank-2R update — over their CUDA-event time, so `frac` is the DMMA-pipe
    utilisation (it agrees with ncu's DMMA-busy).  The reference ledger's rate over the
    same time is `ledger_tflops` (the algorithmic flops of the reference's ZHERK/ZHER2K
    forms; exceeds the DMMA peak because the kernels execute fewer products)."""
    kc_ms = statistics.mean(kern["contract_S"]) + statistics.mean(kern["contract_H"])
    ex = executed_flops(fc, kc_ms, products, n, rows, hpd_rows, joint_rows)
    ledger_tf = fc / (kc_ms / 1e3) / 1e12
    return {
        "bound": "tensor", "achieved": ex["executed_tflops"], "peak": FP64_PEAK_TFLOPS,
        "unit": "TFLOP/s", "frac": ex["executed_frac"], "traffic": traffic,
        "kernel": "contract_kernel (S + H triangular DMMA contractions)",
        "peak_source": "measured FP64 DMMA ceiling, profiles/r01_fp64_peaks.json "
                       "(MEASURED_PEAKS.json has no FP64 entry)",
        "algorithmic_flops_per_step": ex["executed_flops_per_step"],
        "complex_mul": ex["complex_mul"], "h_joint_rows": ex["h_joint_rows"],
        "contract_ms_per_step": round(kc_ms, 4),
        "ledger_flops_per_step": int(fc), "ledger_tflops": round(ledger_tf, 3),
        "kernel_ms": {k: round(statistics.mean(v), 4) for k, v in kern.items() if v},
    }


def kpoint_specs(inst, rank, world):
    """A k-point batch config (C5: 64 seeded k-points, each with its own G-set) is dealt
    round-robin over the ranks and each rank cycles through its share, one k-point per step;
    single-k-point configs give every rank its own seeded k-point of the same crystal."""
    from paper_1602_06589_b200 import configs

    if len(inst.specs) > 1:
        return [inst.specs[i] for i in range(rank, len(inst.specs), world)]
    return [configs.kpoint_variant(inst, rank)]


def measure_kpoint_config(config, steps, warmup, rank, world):
    """Extra key: a k-point config timed like the main line (C5 = BASELINE's k-point batch,
    round-robin over the GPUs); returns a dict for rank 0."""
    import torch

    from paper_1602_06589_b200 import _native, configs
    from paper_1602_06589_b200.pipeline import DeviceSpec, HSPipeline, pack_tmats

    inst = configs.make_instance(config)
    specs = kpoint_specs(inst, rank, world)
    dspecs = [DeviceSpec(x) for x in specs]
    tpack = pack_tmats(inst.tmats)
    pipe = HSPipeline(max(x.n_basis for x in specs), dspecs[0].heights)
    res = None
    for i in range(max(warmup, 3)):
        res = pipe.run(dspecs[i % len(dspecs)], tpack)
    torch.cuda.synchronize()
    ms, kern, ab_ms, res = time_kpoints(pipe, dspecs, tpack, steps, world)
    mask = res["hpd_mask"]
    step_specs = [specs[i % len(specs)] for i in range(steps)]
    flops = sum(configs.nominal_flops(x, mask) for x in step_specs)
    ms_max, tot_flops = max_over_ranks([ms], world)[0], max_over_ranks([flops], world, "sum")[0]
    out = None
    if rank == 0:
        dspec = dspecs[0]
        rows = dspec.rows
        hpd_rows = int(sum(h for h, m in zip(dspec.heights, mask) if m))
        fc = statistics.mean(contract_flops(x.n_basis, rows, hpd_rows) for x in step_specs)
        n_mean = int(round(statistics.mean(x.n_basis for x in step_specs)))
        rl = contraction_roofline(fc, kern, _native.load().hsdla_complex_mul_products(), n_mean,
                                  rows, hpd_rows, joint_rows_of(dspec, tpack, res))
        out = {"workload": workload_name(config, inst), "scaling": "weak",
               "parallelism": f"kpoint-dp{world}",
               "kpoints_per_s": round(world * steps / (ms_max / 1e3), 3),
               "ms_per_kpoint_per_gpu": round(ms_max / steps, 4),
               "tflops": round(tot_flops / (ms_max / 1e3) / 1e12, 4),
               "contract_frac": rl["frac"], "contract_tflops": rl["achieved"]}
    del pipe
    torch.cuda.empty_cache()
    return out


def self_test_p2p(world):
    """P2P panel transport self-test on a small system: the symmetric-memory build must
    agree bitwise with the NCCL gather.  Every rank returns the same verdict."""
    import torch
    import torch.distributed as dist

    from paper_1602_06589_b200 import configs
    from paper_1602_06589_b200.pipeline import DeviceSpec, pack_tmats
    from paper_1602_06589_b200.shard import NcclShardedBuild, P2PShardedBuild

    ok = 1
    try:
        inst = configs.make_instance("C1")
        spec = inst.spec
        dspec, tpack = DeviceSpec(spec), pack_tmats(inst.tmats)
        ref = NcclShardedBuild(spec.n_basis, dspec.heights).run(dspec, tpack)
        p2p = P2PShardedBuild(spec.n_basis, dspec.heights).run(dspec, tpack)
        if ref is not None:
            ok = int(torch.equal(ref[0], p2p[0]) and torch.equal(ref[1], p2p[1]))
    except Exception as e:  # noqa: BLE001 — any failure selects the NCCL transport
        print(f"bench: p2p self-test failed: {e!r}", file=sys.stderr)
        ok = 0
    flag = torch.tensor([ok], device="cuda")
    if world > 1:
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return bool(flag.item())


def measure_panels(config, steps, warmup, rank, world, transport="nccl"):
    """One k-point per step split over all ranks by column panels (SURVEY §8e, C3/C4 strong
    scaling): every rank regenerates A*/B* locally, computes its owned lower tiles; the
    panels reach rank 0 by NCCL send/recv (+ mirror there) or by the contraction epilogue's
    NVLink stores (p2p).  Timed with CUDA events per rank, max over ranks; returns
    (dict for rank 0, sharded-build object, dspec, tpack)."""
    import torch
    import torch.distributed as dist

    from paper_1602_06589_b200 import _native, configs
    from paper_1602_06589_b200.pipeline import DeviceSpec, pack_tmats
    from paper_1602_06589_b200.shard import NcclShardedBuild, P2PShardedBuild

    if transport == "p2p" and not self_test_p2p(world):
        transport = "nccl (p2p self-test failed)"
    inst = configs.make_instance(config)
    spec = inst.spec
    n = spec.n_basis
    dspec = DeviceSpec(spec)
    tpack = pack_tmats(inst.tmats)
    sb = (P2PShardedBuild if transport == "p2p" else NcclShardedBuild)(n, dspec.heights)
    for _ in range(max(warmup, 3)):
        sb.run(dspec, tpack)
    kern = collections.defaultdict(list)
    stream = torch.cuda.current_stream()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            sb.run(dspec, tpack)
            res = sb.last_result
            for k, v in res["kernel_ms"].items():
                kern[k].append(v)
        e1.record(stream)
        torch.cuda.synchronize()
    ms_max = max_over_ranks([e0.elapsed_time(e1)], world)[0]
    mask = res["hpd_mask"]
    flops_step = configs.nominal_flops(spec, mask)
    out = None
    if rank == 0:
        rows = dspec.rows
        hpd_rows = int(sum(h for h, m in zip(dspec.heights, mask) if m))
        fc = contract_flops(n, rows, hpd_rows) / world  # this rank's share of the tiles
        rl = contraction_roofline(fc, kern, _native.load().hsdla_complex_mul_products(), n, rows,
                                  hpd_rows, joint_rows_of(dspec, tpack, res))
        out = {"workload": workload_name(config, inst) + f", split over {world} GPU(s) by "
                                                         "column panels",
               "scaling": "strong", "parallelism": f"panels-{transport.split()[0]}{world}",
               "transport": transport,
               "ms_per_kpoint": round(ms_max / steps, 4),
               "tflops": round(flops_step * steps / (ms_max / 1e3) / 1e12, 4),
               "ledger_flops_per_step": flops_step,
               "contract_frac_rank0": rl["frac"], "contract_tflops_rank0": rl["achieved"],
               "clocks": clk.summary()}
    return out, sb, dspec, tpack, flops_step


def gpu_of(local, args):
    """Device of a local rank: its own GPU; with --backend gloo ranks may share GPUs (the
    multi-rank flow check on a one-GPU box)."""
    import torch

    return local % torch.cuda.device_count() if args.backend == "gloo" else local


def run_ours(args):
    import torch

    from paper_1602_06589_b200 import BuildConfig, _native, configs
    from paper_1602_06589_b200.pipeline import (DeviceSpec, HSPipeline, build_hs, build_hs_many,
                                                pack_tmats)

    rank, world, local = dist_env()
    torch.cuda.set_device(gpu_of(local, args))
    init_dist(world, gpu_of(local, args), args.backend)
    inst = configs.make_instance(args.config)
    specs = kpoint_specs(inst, rank, world)
    spec = specs[0]
    dspecs = [DeviceSpec(x) for x in specs]
    dspec = dspecs[0]
    n = spec.n_basis
    n_cap = max(x.n_basis for x in specs)
    tpack = pack_tmats(inst.tmats)
    pipe = HSPipeline(n_cap, dspec.heights)

    for i in range(max(args.warmup, 3)):
        res = pipe.run(dspecs[i % len(dspecs)], tpack)
    torch.cuda.synchronize()
    mask = res["hpd_mask"]
    rows = dspec.rows
    hpd_rows = int(sum(h for h, m in zip(dspec.heights, mask) if m))
    step_specs = [specs[i % len(specs)] for i in range(args.steps)]
    flops_steps = [configs.nominal_flops(x, mask) for x in step_specs]
    fc_steps = [contract_flops(x.n_basis, rows, hpd_rows) for x in step_specs]

    with ClockSampler(torch.cuda.current_device()) as clk:
        ms, kern, ab_ms, res = time_kpoints(pipe, dspecs, tpack, args.steps, world)
    ms_max = max_over_ranks([ms], world)[0]
    total_flops = max_over_ranks([sum(flops_steps)], world, "sum")[0]
    value = total_flops / (ms_max / 1e3) / 1e12

    # e2e: the public API with host buffers.  build_hs_many = a k-point batch through the
    # pipelined native path: every step uploads its spec (H2D), computes, and copies the
    # full H and S into pinned host memory; k-point i's copies overlap k-point i+1's compute.
    # Also timed: the single synchronous call build_hs (no cross-step overlap).
    bufs = {}
    n_e2e = max(3, args.steps)
    e2e_specs = [specs[i % len(specs)] for i in range(n_e2e)]
    build_hs_many(e2e_specs[:args.warmup], inst.tmats, BuildConfig(), pipeline=pipe,
                  host_buffers=bufs)
    batch_ms = []
    for _ in range(3):  # median of three batches: the host wall clock is noisier than events
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rr = build_hs_many(e2e_specs, inst.tmats, BuildConfig(), pipeline=pipe,
                           host_buffers=bufs)
        torch.cuda.synchronize()
        batch_ms.append((time.perf_counter() - t0) * 1e3 / n_e2e)
    e2e_step_ms = statistics.median(batch_ms)
    h2d = sum(r["h2d_bytes"] for r in rr) / n_e2e
    d2h = sum(r["d2h_bytes"] for r in rr) / n_e2e
    e2e_fl = float(sum(configs.nominal_flops(x, mask) for x in e2e_specs)) / n_e2e
    single_ms = []
    host_out = None
    for i in range(args.warmup + 3):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        h, s, r = build_hs(spec, inst.tmats, BuildConfig(), pipeline=pipe, host_out=host_out)
        torch.cuda.synchronize()
        host_out = (torch.from_numpy(h.base.T), torch.from_numpy(s.base.T))
        if i >= args.warmup:
            single_ms.append((time.perf_counter() - t1) * 1e3)
    dropin = dropin_e2e(spec, inst.tmats, args.warmup)
    e2e_ms, single, dropin_ms = max_over_ranks([e2e_step_ms, statistics.median(single_ms),
                                                dropin["ms"]], world)
    e2e_fl_all = max_over_ranks([e2e_fl], world, "sum")[0]
    e2e_value = e2e_fl_all / (e2e_ms / 1e3) / 1e12
    launches = args.steps * (pipe.launches_per_run(dspec, res)
                             + int(any(res.get("joint_split", [])))
                             + int(res.get("joint_shift", 0.0) > 0))
    clocks = clk.summary()
    del pipe, bufs, host_out, h, s
    torch.cuda.empty_cache()

    extras = {}
    if not args.no_extras and args.config == "C2":
        # BASELINE's scaling configs at this N (the driver's SCALE run covers N = 1, 2, 4, 8):
        # C5 k-points round-robin (weak), C3 one k-point split by column panels (strong).
        # An extra that fails (the N > 1 transports have only met gloo and one-GPU NCCL so far)
        # is reported in its own key; the headline measurement above is already complete and
        # must still be printed.
        try:
            extras["C5_kpoint_batch"] = measure_kpoint_config("C5", max(8, min(args.steps, 64)),
                                                              args.warmup, rank, world)
        except Exception as exc:  # noqa: BLE001
            extras["C5_kpoint_batch"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        try:
            p_out, sb, *_ = measure_panels("C3", max(4, min(args.steps, 16)), args.warmup, rank,
                                           world, args.panel_transport)
            extras["C3_panels"] = p_out
            del sb
        except Exception as exc:  # noqa: BLE001
            extras["C3_panels"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()

    if rank == 0:
        fc = statistics.mean(fc_steps)  # mean per step (k-point batches vary N_G)
        products = _native.load().hsdla_complex_mul_products()
        traffic = None
        tpath = os.path.join(REPO, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                traffic = json.load(f).get("dram_bytes_per_step")
        rl = contraction_roofline(fc, kern, products, n, rows, hpd_rows,
                                  joint_rows_of(dspec, tpack, res), traffic)
        step_ms = ms_max / args.steps
        ex_step = rl["algorithmic_flops_per_step"] / (step_ms / 1e3) / 1e12
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(step_ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": workload_name(args.config, inst),
                "n_basis": n, "rows": rows,
                "ledger_flops_per_step": int(round(total_flops / (world * args.steps))),
                "parallelism": f"kpoint-dp{world}",
                "multi_gpu": ("each GPU builds its own k-point of the same crystal per step "
                              "(k-point parallelism, no collective in the data path)"),
                "l2": "inputs+outputs per step exceed the 126 MB L2 (A,B,UB,Z,XY + H,S); no flush",
            },
            "gpus_active": world,
            "ms_per_kpoint": round(step_ms, 4),
            "kpoints_per_s": round(world * args.steps / (ms_max / 1e3), 2),
            "effective_tflops": round(value / world, 4),
            "effective_note": "value = the reference ledger's flops (predict_flops, builder.py:336-370) "
                              "per second; the kernels execute fewer (DESIGN §3), so this rate is "
                              "not a utilisation — fp64_peak_frac / roofline.frac are",
            "fp64_peak_frac": rl["frac"],
            "step_fp64_frac": round(ex_step / FP64_PEAK_TFLOPS, 4),
            "roofline": {**rl, "ceilings": fp64_ceilings(clocks.get("sm_mhz")),
                         "merged_sh": bool(res.get("merged_sh"))},
            "ab_gen": ab_gen_line(statistics.mean(ab_ms), rows, n, res.get("template_types", 0),
                                  statistics.mean(kern["expand_W"]) if kern.get("expand_W") else None,
                                  statistics.mean(kern["templates"]) if kern.get("templates") else None),
            "e2e": {"value": round(e2e_value, 4), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": round(e2e_ms, 3),
                    "api": "paper_1602_06589_b200.pipeline.build_hs_many (k-point batch: host "
                           "spec per step + T once -> full H, S in pinned host memory per step)",
                    "single_call_ms": round(single, 3),
                    "dropin_ms": round(dropin_ms, 3),
                    "dropin_api": dropin["api"],
                    "dropin_phases_ms": dropin["phases"]},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        line.update({k: v for k, v in extras.items() if v is not None})
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline_sample(args.config, inst)
        print(json.dumps(line), flush=True)


def dropin_e2e(spec, tmats, warmup, reps=3):
    """The reference entry points with host data: compute_AB (flapw.py:201) followed by
    build_all (builder.py:403) returning full H, S in host memory — what a caller of the
    reference sees.  Median of `reps` calls after `warmup` (ms, phase split)."""
    import torch

    import paper_1602_06589_b200 as pkg

    times, ab_t, build_t = [], [], []
    for i in range(warmup + reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        coeffs = pkg.compute_AB(spec)
        t1 = time.perf_counter()
        h, s, _ = pkg.build_all(coeffs, tmats, pkg.BuildConfig())
        t2 = time.perf_counter()
        if i >= warmup:
            times.append((t2 - t0) * 1e3)
            ab_t.append((t1 - t0) * 1e3)
            build_t.append((t2 - t1) * 1e3)
        del h, s, coeffs
    return {"ms": statistics.median(times),
            "phases": {"compute_AB": round(statistics.median(ab_t), 3),
                       "build_all": round(statistics.median(build_t), 3)},
            "api": "paper_1602_06589_b200.compute_AB(spec) + build_all(coeffs, tmats, BuildConfig()) "
                   "-> H, S ComplexDense in host memory (reference flapw.py:201, builder.py:403)"}


def cpu_baseline_sample(config, inst):
    """Bounded CPU sample (~10 s): distinct seeded k-points of the config through the oracle
    port on every host thread; rank 0, N=1 only."""
    from paper_1602_06589_b200 import configs

    _limits = use_all_host_threads()  # noqa: F841
    step, kind, label = cpu_step_fn()
    if kind == "reference":  # numba JIT of the reference's table kernels stays out of the sample
        step(cpu_sample(inst), inst.tmats)
    tot_t = tot_fl = t_ab_sum = t_b_sum = 0.0
    k = 0
    nb = set()
    while k < 30 and (k == 0 or tot_t < 10.0):
        cspec = cpu_sample(configs.Instance(inst.cfg, [configs.kpoint_variant(inst, k)],
                                            inst.tmats, inst.min_abs_wronskian))
        nb.add(cspec.n_basis)
        dt, fl, t_ab, t_build = step(cspec, inst.tmats)
        tot_t, tot_fl, t_ab_sum, t_b_sum, k = (tot_t + dt, tot_fl + fl, t_ab_sum + t_ab,
                                               t_b_sum + t_build, k + 1)
    return {
        "value": round(tot_fl / tot_t / 1e12, 4), "unit": UNIT, "cores": host_threads(),
        "kind": kind,
        "sample": f"{k} distinct seeded k-point(s) of {config} (N_G {min(nb)}-{max(nb)}), "
                  f"{tot_t:.1f} s: {label.split(' compute_AB')[0]} compute_AB {t_ab_sum / k:.2f} s "
                  f"+ build_all {t_b_sum / k:.2f} s per k-point (scipy OpenBLAS)",
    }


def run_panels(args):
    """`--mode panels`: the line is one k-point per step split over all ranks (strong scaling)."""
    import torch

    from paper_1602_06589_b200.pipeline import DeviceSpec

    rank, world, local = dist_env()
    torch.cuda.set_device(gpu_of(local, args))
    init_dist(world, gpu_of(local, args), args.backend)
    out, sb, dspec, tpack, flops_step = measure_panels(args.config, args.steps, args.warmup,
                                                       rank, world, args.panel_transport)
    # e2e: spec upload + sharded build + full H, S read back to pinned host on rank 0
    n = dspec.n_basis
    spec = __import__("paper_1602_06589_b200").configs.make_instance(args.config).spec
    hh = torch.empty((n, n), dtype=torch.complex128, pin_memory=True) if rank == 0 else None
    hs = torch.empty((n, n), dtype=torch.complex128, pin_memory=True) if rank == 0 else None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = sb.run(DeviceSpec(spec), tpack)
        if res is not None:
            hh.copy_(res[0], non_blocking=True)
            hs.copy_(res[1], non_blocking=True)
        torch.cuda.synchronize()
    e2e = max_over_ranks([(time.perf_counter() - t0) * 1e3 / args.steps], world)[0]
    if rank == 0:
        line = {
            "metric": METRIC, "value": out["tflops"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": out["ms_per_kpoint"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": out["workload"], "n_basis": n, "rows": dspec.rows,
                       "ledger_flops_per_step": flops_step, "parallelism": out["parallelism"],
                       "l2": "operands and H, S exceed the 126 MB L2; no flush"},
            "gpus_active": world,
            "fp64_peak_frac": out["contract_frac_rank0"],
            "panels": out,
            "e2e": {"value": round(flops_step / (e2e / 1e3) / 1e12, 4), "unit": UNIT,
                    "h2d_bytes_per_step": int(dspec.h2d_bytes), "d2h_bytes_per_step": 32 * n * n,
                    "ms_per_step": round(e2e, 3),
                    "api": f"paper_1602_06589_b200.shard.{type(sb).__name__}.run + D2H of H, S"},
            "gpu_launches": args.steps * (sb.pipe.launches_per_run(dspec, sb.last_result)
                                          + (2 if world > 1 else 0)),
            "clocks": out["clocks"],
        }
        print(json.dumps(line), flush=True)


def run_dry(args):
    """Launcher check without a GPU (gloo): every rank reports the work it would take —
    its k-points of the C5 batch and its column panels of C3 — and rank 0 prints one line."""
    import socket

    import torch.distributed as dist

    from paper_1602_06589_b200.shard import kpoints_for_rank, owned_panels

    rank, world, _ = dist_env()
    init_dist(world, 0, backend="gloo")
    mine = {"rank": rank, "host": socket.gethostname(), "pid": os.getpid(),
            "c5_kpoints": kpoints_for_rank(64, world, rank),
            "c3_panels": len(owned_panels(7994, world, rank))}
    got = [None] * world
    if world > 1:
        dist.all_gather_object(got, mine)
    else:
        got = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "gpus_active": world,
                          "steps": args.steps, "warmup": args.warmup,
                          "config": {"workload": args.config}, "ranks": got}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` started without torchrun: re-launch this script under
    torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous) and return its
    exit code; rank 0's JSON line is the output."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    if not args.dry_run and args.backend != "gloo":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench: --gpus {args.gpus} but only {have} CUDA device(s) visible",
                  file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        run_dry(args)
    elif args.mode == "panels":
        run_panels(args)
    else:
        run_ours(args)
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
