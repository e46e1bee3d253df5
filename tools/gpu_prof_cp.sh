#!/bin/bash
# One full ncu capture (source-level) of the S contraction launch (cp.async kernel).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
CFG=${CFG:-C2}
python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_short.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"contract" -s 4 -c 1 \
    -o gpurun_out/prof_cpS_$CFG python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
