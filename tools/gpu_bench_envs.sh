#!/bin/bash
# bench.py kernel breakdown under several environment settings, one box:
# BENCH_ENVS="A=1,B=2 C=3" (commas -> spaces), CFGS="C2 C3".
cd "$GRAFT_REPO_ROOT"
export PYTHONDONTWRITEBYTECODE=1
for c in ${CFGS:-C2}; do
  for e in $BENCH_ENVS; do
    echo -n "$c $e: "; env ${e//,/ } timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step'])"
  done
done
