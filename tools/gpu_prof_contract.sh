#!/bin/bash
# tests, bench, then one full ncu capture of the S contraction launch.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
CFG=${CFG:-C2}
timeout 600 python bench.py --config $CFG > gpurun_out/bench_$CFG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$CFG.log
cat gpurun_out/bench_$CFG.log
python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_short.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"contract" -s 4 -c 1 \
    -o gpurun_out/prof_contractS_$CFG python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
