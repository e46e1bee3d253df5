#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for v in 64 96; do
  HSDLA_APPLY_TILE=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_a$v.log 2>&1
  echo -n "apply tile $v rc=$? "; tail -1 gpurun_out/bench_a$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step'])"
done
