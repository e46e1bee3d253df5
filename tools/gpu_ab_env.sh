#!/bin/bash
# A (tools/libA.so, default env) vs B (tools/libB.so with $B_ENV) on one box.
cd "$GRAFT_REPO_ROOT"
cp paper_1602_06589_b200/libhsdla_b200.so /tmp/lib_orig.so
for r in 1 2; do
  cp tools/libA.so paper_1602_06589_b200/libhsdla_b200.so
  echo -n "A "; python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms'])"
  cp tools/libB.so paper_1602_06589_b200/libhsdla_b200.so
  echo -n "B "; env $B_ENV python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms'])"
done
env $B_ENV python tools/contract_loop_probe.py | grep -E "16384|8000"
cp /tmp/lib_orig.so paper_1602_06589_b200/libhsdla_b200.so
