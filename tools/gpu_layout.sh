#!/bin/bash
# Parity + A/B of the cp.async shared-memory layouts (HSDLA_CP_LAYOUT).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_layout.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_layout.log
for lay in ${LAYOUTS:-xor pair xor pair}; do
  HSDLA_CP_LAYOUT=$lay timeout 300 python bench.py --config ${CFG:-C2} --no-cpu-baseline > gpurun_out/bench_$lay.log 2>&1
  echo "layout=$lay"; tail -1 gpurun_out/bench_$lay.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value'])"
done
