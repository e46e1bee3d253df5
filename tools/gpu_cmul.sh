#!/bin/bash
# Three- vs four-product complex multiply in the triangular contractions (HSDLA_CMUL), one box:
# parity tests under the default, then bench C2/C3 lines for both.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for c in C2 C3; do
  for m in 4 3 4 3; do
    echo -n "$c cmul=$m "; HSDLA_CMUL=$m timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step'])"
  done
done
