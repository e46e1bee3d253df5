#!/bin/bash
# bench (plain) then ncu launch list + one full capture of the contraction kernel.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
CFG=${CFG:-C2}
python bench.py --config $CFG --steps 30 --warmup 3 > gpurun_out/bench_$CFG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$CFG.log
cat gpurun_out/bench_$CFG.log
python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
    python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
if [ -n "$FULL" ]; then
ncu --set full --clock-control none --import-source on -k regex:contract_kernel -s 8 -c 2 \
    -o gpurun_out/prof_contract_$CFG python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
fi
