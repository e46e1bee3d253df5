#!/bin/bash
# Full evidence pass: GPU tests, smoke, bench C2 (default) + C3/C4/C5, ncu launch list,
# one ncu --set full capture of the S contraction, DRAM traffic of the contractions.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_C2.log 2>&1; echo "bench C2 rc=$?"
tail -1 gpurun_out/bench_C2.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
tail -1 gpurun_out/bench_ref.log
for c in C3 C4 C5 C2NS C2IND; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_$c.log | cut -c1-400
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_short.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"contract" -s 4 -c 1 \
    -o gpurun_out/prof_contractS_C2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"contract" --csv --log-file gpurun_out/traffic_C2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_t.log 2>&1
echo "ncu traffic rc=$?"
