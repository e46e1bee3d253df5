#!/bin/bash
# Main-loop probe for both complex-multiply variants, then one ncu --set full capture of the
# S contraction (C2) under the default (three-product) kernel.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
for m in 4 3; do echo "cmul=$m"; HSDLA_CMUL=$m timeout 300 python tools/contract_loop_probe.py; done
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_short.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"contract" -s 4 -c 1 \
    -o gpurun_out/prof_g3_S_C2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
