#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
HSDLA_CONTRACT=tma timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_tma.log 2>&1; echo "pytest tma rc=$?" >> gpurun_out/pytest_tma.log
tail -25 gpurun_out/pytest_tma.log
for v in auto tma; do
  HSDLA_CONTRACT=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
  echo -n "$v rc=$? "; tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step'])"
done
