#!/bin/bash
# tests + A/B comparison of contraction variants on the bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for v in 16 32; do
  HSDLA_WARP_COLS=$v timeout 600 python bench.py --config ${CFG:-C2} --no-cpu-baseline > gpurun_out/bench_w$v.log 2>&1
  echo "variant $v rc=$?"; cat gpurun_out/bench_w$v.log | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step'])"
done
