#!/bin/bash
# A/B two library builds (tools/libA.so, tools/libB.so): bench value + e2e steady interval.
cd "$GRAFT_REPO_ROOT"
cp paper_1602_06589_b200/libhsdla_b200.so /tmp/lib_orig.so
for r in 1 2; do
for v in A B; do
  cp tools/lib$v.so paper_1602_06589_b200/libhsdla_b200.so
  echo -n "$v "; python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step'])"
  python tools/e2e_probe.py C2 | tail -1
done; done
cp /tmp/lib_orig.so paper_1602_06589_b200/libhsdla_b200.so
