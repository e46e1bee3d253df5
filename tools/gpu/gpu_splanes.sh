# SP (shared-memory sum planes per chunk) vs default contraction: parity with SP on, then
# bench lines back to back (alternating) on C2 / C3.
mkdir -p gpurun_out/sp
HSDLA_SPLANES=1 python -m pytest tests/test_gpu_contracts.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_golden_big.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/sp/pytest_sp.log
for r in 1 2; do
  for v in 0 1; do
    HSDLA_SPLANES=$v python bench.py --steps 20 --no-extras --no-cpu-baseline > gpurun_out/sp/C2_sp${v}_r$r.json 2>/dev/null
  done
done
for v in 0 1; do
  HSDLA_SPLANES=$v python bench.py --config C3 --steps 3 --no-extras --no-cpu-baseline > gpurun_out/sp/C3_sp$v.json 2>/dev/null
done
