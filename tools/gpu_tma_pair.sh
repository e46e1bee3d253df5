#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONDONTWRITEBYTECODE=1
HSDLA_CONTRACT=tma timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
for r in 1 2; do
for m in "auto 1" "auto 0" "tma 1" "tma 0"; do
  set -- $m
  echo -n "contract=$1 pair=$2 "
  HSDLA_CONTRACT=$1 HSDLA_TMA_PAIR=$2 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
done; done
