#!/bin/bash
# contract_loop_probe under several environment settings: PROBE_ENVS="A=1,B=2 C=3" (commas -> spaces).
cd "$GRAFT_REPO_ROOT"
export PYTHONDONTWRITEBYTECODE=1
for e in $PROBE_ENVS; do
  echo "== $e"; env ${e//,/ } timeout 300 python tools/contract_loop_probe.py
done
