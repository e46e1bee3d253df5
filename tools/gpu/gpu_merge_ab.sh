# A/B of the merged S + H contraction launch (HSDLA_MERGE_SH) on C2 and C5, plus the GPU suite.
set -x
mkdir -p gpurun_out/mab
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/mab/pytest.log
for rep in 1 2; do
  for m in 1 0; do
    HSDLA_MERGE_SH=$m python bench.py --steps 30 --no-extras --no-cpu-baseline > gpurun_out/mab/C2_m${m}_$rep.json 2> gpurun_out/mab/C2_m${m}_$rep.err
    HSDLA_MERGE_SH=$m python bench.py --config C5 --steps 30 --no-extras --no-cpu-baseline > gpurun_out/mab/C5_m${m}_$rep.json 2> gpurun_out/mab/C5_m${m}_$rep.err
  done
done
for m in 1 0; do
  HSDLA_MERGE_SH=$m python bench.py --config C3 --steps 5 --no-extras --no-cpu-baseline > gpurun_out/mab/C3_m${m}.json 2> gpurun_out/mab/C3_m${m}.err
done
