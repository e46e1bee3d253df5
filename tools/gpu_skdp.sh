#!/bin/bash
# A/B of data-parallel waves ahead of stream-K (HSDLA_SK_DP) + parity + DRAM traffic.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_skdp.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_skdp.log
for dp in 0 1 0 1; do
  HSDLA_SK_DP=$dp timeout 300 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_dp$dp.log 2>&1
  echo "dp=$dp"; tail -1 gpurun_out/bench_dp$dp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['value'])"
done
for dp in 0 1; do
HSDLA_SK_DP=$dp ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"contract" --csv --log-file gpurun_out/traffic_dp$dp.csv \
    python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dp$dp.log 2>&1
echo "ncu dp=$dp rc=$?"
done
