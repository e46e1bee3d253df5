"""Benchmark of the muffin-tin H/S setup (FLAPW, HSDLA) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one k-point of the BASELINE configuration through the hot path
(A/B generation + Cholesky/T application + the S and H triangular DMMA contractions
with the fused Hermitian mirror), inputs (SystemSpec, T blocks) resident in HBM.
The metric is BASELINE.json's: H+S setup time per k-point and FP64 TFLOP/s over the
reference's nominal FLOP ledger (`builder.py:336-370`), as a fraction of the measured
FP64 DMMA peak.  Multi-GPU: one process per GPU (torchrun), each rank builds its own
k-point (k-point parallelism, weak scaling, no collective in the data path); the
time is the max over ranks.  `--impl reference` times the CPU oracle port (numpy +
the same scipy/OpenBLAS routines the reference's optimized backend calls) on the
host cores, rank 0 only.  Prints one JSON line.
"""
from __future__ import annotations

import argparse
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
                        "panels: ONE k-point split over all GPUs by column panels, tiles "
                        "stored into rank 0's H/S over NVLink peer memory (strong scaling)")
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
    spec = cpu_sample(inst)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_oracle_step(spec, inst.tmats)
    times, flops = [], 0
    t_start = time.perf_counter()
    for _ in range(args.steps):
        dt, fl, _, _ = cpu_oracle_step(spec, inst.tmats)
        times.append(dt)
        flops = fl
        if time.perf_counter() - t_start > 150:  # keep the arm within a few minutes
            break
    total = sum(times)
    value = flops * len(times) / total / 1e12
    sample = (f"{len(times)} full k-point(s) of {args.config}" +
              (f" truncated to N_G={spec.n_basis}" if spec.n_basis < inst.spec.n_basis else
               f" (N_G={spec.n_basis})") + ": oracle compute_AB + build_all (scipy OpenBLAS)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / len(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": (f"{args.config} (BASELINE.json configs[{int(args.config[1]) - 1}])"
                                if len(args.config) == 2 else f"{args.config} (not a BASELINE config)"),
                   "n_basis": spec.n_basis, "rows": int(sum((l + 1) ** 2 for l in spec.l_sph))},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": host_threads(),
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
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


def ab_gen_line(ms, rows, n):
    """A/B generation against the HBM-write roofline: the generator writes A*,
    B* and ||udot|| B* (48 R N bytes; the reference's Bytes_AB counts A*, B* = 32 R N)."""
    peak, src = hbm_peak_gbs()
    written = 48 * rows * n
    gbs = written / (ms / 1e3) / 1e9
    return {"ms": round(ms, 4), "bytes_written": written, "bytes_ab_ref": 32 * rows * n,
            "achieved_gbs": round(gbs, 1), "peak_gbs": peak, "peak_source": src,
            "frac": round(gbs / peak, 4)}


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
            "note": "achieved/frac count SURVEY 8(d)'s ledger flops (the reference algorithm); the "
                    "kernels execute fewer (three-product multiply, joint T factor for H), so frac "
                    "can exceed 1; executed_frac is the DMMA-pipe utilisation"}


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


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1602_06589_b200 import BuildConfig, _native, configs
    from paper_1602_06589_b200.pipeline import (DeviceSpec, HSPipeline, build_hs, build_hs_many,
                                                pack_tmats)

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    inst = configs.make_instance(args.config)
    # A k-point batch config (C5: 64 seeded k-points, each with its own G-set) is dealt
    # round-robin over the ranks and each rank cycles through its share, one k-point per step;
    # single-k-point configs give every rank its own seeded k-point of the same crystal.
    specs = ([inst.specs[i] for i in range(rank, len(inst.specs), world)]
             if len(inst.specs) > 1 else [configs.kpoint_variant(inst, rank)])
    spec = specs[0]
    dspecs = [DeviceSpec(x) for x in specs]
    dspec = dspecs[0]
    n = spec.n_basis
    n_cap = max(x.n_basis for x in specs)
    tpack = pack_tmats(inst.tmats)
    pipe = HSPipeline(n_cap, dspec.heights)
    stream = torch.cuda.current_stream()

    for i in range(max(args.warmup, 3)):
        res = pipe.run(dspecs[i % len(dspecs)], tpack)
    torch.cuda.synchronize()
    mask = res["hpd_mask"]
    rows = dspec.rows
    hpd_rows = int(sum(h for h, m in zip(dspec.heights, mask) if m))
    step_specs = [specs[i % len(specs)] for i in range(args.steps)]
    flops_steps = [configs.nominal_flops(x, mask) for x in step_specs]
    flops_step = flops_steps[0]
    fc_steps = [contract_flops(x.n_basis, rows, hpd_rows) for x in step_specs]
    fc = fc_steps[0]

    kern = {"contract_S": [], "contract_H": [], "apply_Z": [], "apply_XY": []}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        # k-points back to back through the pipelined native path: step i+1 is enqueued
        # before step i is collected, so host-side enqueue never idles the GPU.
        prev = None
        ab_ms = []

        def collect(ticket):
            r = pipe.finish(ticket)
            for k, v in r["kernel_ms"].items():
                kern[k].append(v)
            ab_ms.append(r["ms"]["setup"])  # A/B generation (T preparation reused)

        for i in range(args.steps):
            ticket = pipe.run_async(dspecs[i % len(dspecs)], tpack)
            if prev is not None:
                collect(prev)
            prev = ticket
        e1.record(stream)
        collect(prev)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], device="cuda")
    fl_t = torch.tensor([float(sum(flops_steps))], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(fl_t, op=dist.ReduceOp.SUM)
    ms_max = float(ms_t.item())
    total_flops = float(fl_t.item())
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
    e2e_fl = torch.tensor([float(sum(configs.nominal_flops(x, mask) for x in e2e_specs)) / n_e2e],
                          device="cuda", dtype=torch.float64)
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
    e2e_t = torch.tensor([e2e_step_ms, statistics.median(single_ms)], device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(e2e_fl, op=dist.ReduceOp.SUM)
    e2e_value = float(e2e_fl.item()) / (float(e2e_t[0].item()) / 1e3) / 1e12

    if rank == 0:
        kc_ms = statistics.mean(kern["contract_S"]) + statistics.mean(kern["contract_H"])
        fc = statistics.mean(fc_steps)  # mean per step (k-point batches vary N_G)
        achieved = fc / (kc_ms / 1e3) / 1e12
        products = _native.load().hsdla_complex_mul_products()
        joint_rows = joint_rows_of(dspec, tpack, res)
        traffic = None
        tpath = os.path.join(REPO, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                traffic = json.load(f).get("dram_bytes_per_step")
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": (f"{args.config}: N_G={n}, N_A={spec.n_atoms}, N_L={int(dspec.heights[0])}, "
                             f"R={rows}, one k-point per GPU per step" if len(inst.specs) == 1 else
                             f"{args.config}: {len(inst.specs)} k-points (N_G "
                             f"{min(x.n_basis for x in inst.specs)}-{max(x.n_basis for x in inst.specs)}), "
                             f"N_A={spec.n_atoms}, N_L={int(dspec.heights[0])}, R={rows}; dealt "
                             f"round-robin over the GPUs, each cycling through its share, one "
                             f"k-point per GPU per step"),
                "n_basis": n, "rows": rows,
                "ledger_flops_per_step": int(round(total_flops / (world * args.steps))),
                "parallelism": f"kpoint-dp{world}",
                "l2": "inputs+outputs per step exceed the 126 MB L2 (A,B,UB,Z,XY + H,S); no flush",
            },
            "ms_per_kpoint": round(ms_max / args.steps, 4),
            "kpoints_per_s": round(world * args.steps / (ms_max / 1e3), 2),
            "fp64_peak_frac": round(value / world / FP64_PEAK_TFLOPS, 4),
            "roofline": {
                "bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                "traffic": traffic,
                "kernel": "contract_kernel (S + H triangular DMMA contractions)",
                "peak_source": "measured FP64 DMMA ceiling, profiles/r01_fp64_peaks.json "
                               "(MEASURED_PEAKS.json has no FP64 entry)",
                "ceilings": fp64_ceilings(clk.summary().get("sm_mhz")),
                "algorithmic_flops_per_step": fc,
                **executed_flops(fc, kc_ms, products, n, rows, hpd_rows, joint_rows,
                                 joint_rows_of(dspec, tpack, res, hpd_only=True)),
                "kernel_ms": {k: round(statistics.mean(v), 4) for k, v in kern.items()},
            },
            "ab_gen": ab_gen_line(statistics.mean(ab_ms), rows, n),
            "e2e": {"value": round(e2e_value, 4), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": round(float(e2e_t[0].item()), 3),
                    "api": "paper_1602_06589_b200.pipeline.build_hs_many (k-point batch: host "
                           "spec per step + T once -> full H, S in pinned host memory per step)",
                    "single_call_ms": round(float(e2e_t[1].item()), 3)},
            "gpu_launches": args.steps * (pipe.launches_per_run(dspec)
                                          + int(any(res.get("joint_split", [])))
                                          + int(res.get("joint_shift", 0.0) > 0)),
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline and world == 1:
            _limits = use_all_host_threads()  # noqa: F841
            # bounded sample: k-points of the config until ~10 s of CPU work (at most 30)
            cspec = cpu_sample(inst)
            tot_t = tot_fl = t_ab_sum = t_b_sum = 0.0
            k = 0
            while k < 30 and (k == 0 or tot_t < 10.0):
                dt, fl, t_ab, t_build = cpu_oracle_step(cspec, inst.tmats)
                tot_t, tot_fl, t_ab_sum, t_b_sum, k = (tot_t + dt, tot_fl + fl, t_ab_sum + t_ab,
                                                       t_b_sum + t_build, k + 1)
            line["cpu_baseline"] = {
                "value": round(tot_fl / tot_t / 1e12, 4), "unit": UNIT, "cores": host_threads(),
                "kind": "port",
                "sample": f"{k} k-point(s) of {args.config} (N_G={cspec.n_basis}), {tot_t:.1f} s: "
                          f"oracle compute_AB {t_ab_sum / k:.2f} s + build_all {t_b_sum / k:.2f} s "
                          f"per k-point (scipy OpenBLAS)",
            }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_panels(args):
    """One k-point per step, column panels over all ranks (SURVEY §8e, C3/C4 strong scaling):
    every rank regenerates A*/B* locally, computes its owned lower tiles and stores them and
    their mirror straight into rank 0's symmetric-memory H and S (shard.P2PShardedBuild)."""
    import torch
    import torch.distributed as dist

    from paper_1602_06589_b200 import _native, configs
    from paper_1602_06589_b200.pipeline import DeviceSpec, pack_tmats
    from paper_1602_06589_b200.shard import P2PShardedBuild

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if "MASTER_ADDR" not in os.environ:  # single process without torchrun
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]),
                              RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    inst = configs.make_instance(args.config)
    spec = inst.spec
    n = spec.n_basis
    dspec = DeviceSpec(spec)
    tpack = pack_tmats(inst.tmats)
    sb = P2PShardedBuild(n, dspec.heights)
    out = None
    for _ in range(max(args.warmup, 3)):
        out = sb.run(dspec, tpack)
    kern = {"contract_S": [], "contract_H": [], "apply_Z": [], "apply_XY": []}
    stream = torch.cuda.current_stream()
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            res = sb.pipe.run(dspec, tpack)
            torch.cuda.synchronize()
            dist.barrier()
            for k, v in res["kernel_ms"].items():
                kern[k].append(v)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    mask = res["hpd_mask"]
    flops_step = configs.nominal_flops(spec, mask)
    value = flops_step * args.steps / (float(ms.item()) / 1e3) / 1e12
    # e2e: spec upload + sharded build + full H, S read back to pinned host on rank 0
    hh = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
    hs = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = sb.run(DeviceSpec(spec), tpack)
        if out is not None:
            hh.copy_(out[0], non_blocking=True)
            hs.copy_(out[1], non_blocking=True)
            torch.cuda.synchronize()
    e2e = torch.tensor([(time.perf_counter() - t0) * 1e3 / args.steps], device="cuda")
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    if rank == 0:
        rows = dspec.rows
        hpd_rows = int(sum(h for h, m in zip(dspec.heights, mask) if m))
        kc = statistics.mean(kern["contract_S"]) + statistics.mean(kern["contract_H"])
        fc = contract_flops(n, rows, hpd_rows) / world  # this rank's share of the tiles
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(float(ms.item()) / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: N_G={n}, R={rows}, one k-point split over "
                                   f"{world} GPU(s) by column panels",
                       "n_basis": n, "rows": rows, "ledger_flops_per_step": flops_step,
                       "parallelism": f"panels-p2p{world}",
                       "l2": "operands and H, S exceed the 126 MB L2; no flush"},
            "fp64_peak_frac": round(value / world / FP64_PEAK_TFLOPS, 4),
            "roofline": {"bound": "tensor", "achieved": round(fc / (kc / 1e3) / 1e12, 3),
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": round(fc / (kc / 1e3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                         "traffic": None,
                         **executed_flops(fc, kc, _native.load().hsdla_complex_mul_products(),
                                          n, rows, hpd_rows, joint_rows_of(dspec, tpack, res),
                                          joint_rows_of(dspec, tpack, res, hpd_only=True)),
                         "kernel_ms": {k: round(statistics.mean(v), 4) for k, v in kern.items()}},
            "e2e": {"value": round(flops_step / (float(e2e.item()) / 1e3) / 1e12, 4), "unit": UNIT,
                    "h2d_bytes_per_step": int(dspec.h2d_bytes), "d2h_bytes_per_step": 32 * n * n,
                    "ms_per_step": round(float(e2e.item()), 3),
                    "api": "paper_1602_06589_b200.shard.P2PShardedBuild.run + D2H of H, S"},
            "gpu_launches": args.steps * (sb.pipe.launches_per_run(dspec)
                                          + int(any(res.get("joint_split", [])))
                                          + int(res.get("joint_shift", 0.0) > 0)),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "panels":
        run_panels(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
