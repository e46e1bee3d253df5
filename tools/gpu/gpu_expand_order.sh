# Expansion grid order by atom count: template-path parity, C2 launch list, bench lines.
mkdir -p gpurun_out/eo
python -m pytest tests/test_gpu_joint.py tests/test_gpu_parity.py tests/test_gpu_golden_big.py tests/test_gpu_edges.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/eo/pytest.log
CMD="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"expand" -c 8 --csv --log-file gpurun_out/eo/launches_C2.csv $CMD > /dev/null 2>&1
for c in C2 C3 C4; do
  python bench.py --config $c --steps 3 --no-extras --no-cpu-baseline > gpurun_out/eo/$c.json 2>/dev/null
done
