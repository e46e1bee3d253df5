# Rolled l-loop for the per-type template generator (HSDLA_AB_ROLL) vs unrolled; parity.
mkdir -p gpurun_out/ar
python -m pytest tests/test_gpu_joint.py tests/test_gpu_parity.py tests/test_gpu_golden_big.py tests/test_gpu_edges.py tests/test_gpu_special.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/ar/pytest.log
for r in 1 2; do
  for v in 0 1; do
    HSDLA_AB_ROLL=$v python bench.py --steps 20 --no-extras --no-cpu-baseline > gpurun_out/ar/C2_${v}_r$r.json 2>/dev/null
    HSDLA_AB_ROLL=$v python bench.py --config C5 --steps 5 --no-extras --no-cpu-baseline > gpurun_out/ar/C5_${v}_r$r.json 2>/dev/null
  done
done
