set -x
mkdir -p gpurun_out/single2
python -m pytest tests/test_gpu_contracts.py tests/test_gpu_fullsize.py tests/test_gpu_golden_big.py -m gpu -x -q 2>&1 | tail -5 > gpurun_out/single2/pytest.log
for m in 1 0; do
HSDLA_MERGE_SH=$m python tools/copy_timeline.py C2 > gpurun_out/single2/timeline_m$m.txt 2>&1
done
python bench.py --steps 20 --no-extras --no-cpu-baseline > gpurun_out/single2/C2.json 2> gpurun_out/single2/C2.err
HSDLA_MERGE_SH=0 python bench.py --steps 20 --no-extras --no-cpu-baseline > gpurun_out/single2/C2_m0.json 2> gpurun_out/single2/C2_m0.err
