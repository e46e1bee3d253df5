#!/bin/bash
# tests + smoke + bench + ncu launch list + full capture of ab_kernel and tprep.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
cat gpurun_out/smoke.log
CFG=${CFG:-C2}
timeout 600 python bench.py --config $CFG > gpurun_out/bench_$CFG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$CFG.log
cat gpurun_out/bench_$CFG.log
python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
    python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"ab_kernel|tprep" -s 2 -c 2 \
    -o gpurun_out/prof_ab_$CFG python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
