#!/bin/bash
# tests + A/B comparison of contraction variants on the bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for pad in 0 1; do for v in 32 16; do
  HSDLA_SMEM_PAD=$pad HSDLA_WARP_COLS=$v timeout 600 python bench.py --config ${CFG:-C2} --no-cpu-baseline > gpurun_out/bench_w${v}_p$pad.log 2>&1
  echo -n "pad $pad warpcols $v rc=$? "; cat gpurun_out/bench_w${v}_p$pad.log | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step'])"
done; done; done
