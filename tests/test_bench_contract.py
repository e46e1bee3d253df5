"""bench.py's output contract on CPU: the reference arm (`--impl reference`: the unmodified
reference package from baseline/_ref where it is installed, else the oracle port, timed on the
host) prints one JSON line with the driver's keys; the GPU arm's helpers
(ledger flops, FP64 ceilings, A/B-generation roofline) compute what DESIGN.md says."""
import json
import os
import subprocess
import sys

from conftest import REPO


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "TFLOP/s" and d["higher_is_better"] is True
    have_ref = os.path.exists(os.path.join(REPO, "baseline", "_ref", "hsdla", "__init__.py"))
    assert d["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["kind"] == ("reference" if have_ref else "port")
    assert ("oracle_port" in d) == have_ref
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_port_fallback():
    """Without the reference package (forced here) the arm is the oracle port."""
    env = dict(os.environ, HSDLA_BENCH_CPU_ARM="port")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=REPO, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["cpu_baseline"]["kind"] == "port" and "oracle_port" not in d and d["value"] > 0


def test_bench_helpers():
    sys.path.insert(0, REPO)
    import bench

    n, r = 3000, 1296
    assert bench.contract_flops(n, r, r) == 16 * r * n * n + 4 * r * n * n
    assert bench.contract_flops(n, r, 0) == 24 * r * n * n
    c = bench.fp64_ceilings(1965.0)
    assert c["dmma_peak_boost_tflops"] == 37.2
    assert abs(c["dmma_peak_at_measured_clock_tflops"] - 37.22) < 0.01
    g = bench.ab_gen_line(0.1, r, n)
    assert g["bytes_written"] == 48 * r * n and 0 < g["frac"] < 1


def test_executed_flops_accounting():
    """Executed DMMA work: S (K = 2R) + H with joint T sets (K = 2R) is 16 R N^2 complex-MAC
    flops; with the reference forms H adds ZHER2K (8 R N^2) + ZHERK or the lower half of the
    ZGEMM (4 R N^2 each).  Three products: x 3/4."""
    sys.path.insert(0, REPO)
    import bench

    n, r = 3000, 1296
    fc = bench.contract_flops(n, r, r)
    joint = bench.executed_flops(fc, 1.0, 3, n, r, r, r)
    assert joint["executed_flops_per_step"] == 16 * r * n * n * 3 // 4
    ref = bench.executed_flops(fc, 1.0, 4, n, r, r, 0)
    assert ref["executed_flops_per_step"] == fc  # four products, reference forms: the ledger
    # non-HPD reference-form rows: the kernel's A^H X lands in the lower triangle only
    mixed = bench.executed_flops(fc, 1.0, 4, n, r, 600, 300)
    assert mixed["executed_flops_per_step"] == (8 * r + 8 * 300 + 12 * (r - 300)) * n * n
    nonhpd = bench.executed_flops(bench.contract_flops(n, r, 0), 1.0, 4, n, r, 0, 0)
    assert nonhpd["executed_flops_per_step"] == 20 * r * n * n

    # shifted joint form: joint rows that are not HPD
    ind = bench.executed_flops(fc, 1.0, 4, n, r, 0, r, 0)
    assert ind["executed_flops_per_step"] == 16 * r * n * n


def test_gpus_flag_spawns_ranks_dry_run():
    """`bench.py --gpus 2` without torchrun re-launches itself with two ranks (the driver calls
    it that way); the gloo dry run shows both ranks ran and dealt the work round-robin."""
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2",
                          "--dry-run", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=REPO,
                         env={k: v for k, v in os.environ.items()
                              if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpus_active"] == 2
    assert sorted(r["rank"] for r in d["ranks"]) == [0, 1]
    assert len({r["pid"] for r in d["ranks"]}) == 2
    ks = sorted(k for r in d["ranks"] for k in r["c5_kpoints"])
    assert ks == list(range(64))


def test_workload_names_match_between_arms():
    sys.path.insert(0, REPO)
    import bench
    from paper_1602_06589_b200 import configs

    for c in ("C1", "C2", "C5"):
        name = bench.workload_name(c, configs.make_instance(c))
        assert name.startswith(c) and "BASELINE.json configs[" in name


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_two_ranks_gloo_on_one_gpu(cuda):
    """The N > 1 bench flow end to end on a one-GPU box: `--gpus 2` spawns two ranks (gloo,
    sharing the GPU), each builds its own C2 k-point, C5 k-points are dealt round-robin and one
    C3 k-point is split by column panels and gathered to rank 0 (host-staged over gloo: the
    NCCL transport of the 8-GPU box is the same gather on device memory); times are the max over
    ranks.  Checks the line's shape, not speed (the ranks time-slice one GPU)."""
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2",
                          "--backend", "gloo", "--steps", "2", "--warmup", "1",
                          "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=1200, cwd=REPO,
                         env={k: v for k, v in os.environ.items()
                              if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpus_active"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"] == "kpoint-dp2"
    assert d["C5_kpoint_batch"]["parallelism"] == "kpoint-dp2"
    assert d["C5_kpoint_batch"]["kpoints_per_s"] > 0
    assert d["C3_panels"]["parallelism"] == "panels-nccl2" and d["C3_panels"]["tflops"] > 0
