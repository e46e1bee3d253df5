#!/bin/bash
# bench (plain) + ncu DRAM traffic per contraction launch (one bench step after warm-up).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
CFG=${CFG:-C2}
timeout 600 python bench.py --config $CFG > gpurun_out/bench_$CFG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$CFG.log
tail -2 gpurun_out/bench_$CFG.log
python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_t.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"contract" --csv --log-file gpurun_out/traffic_$CFG.csv \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_t.log 2>&1
echo "ncu rc=$?"
