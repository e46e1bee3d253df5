# A/B of the single fused expansion pass (HSDLA_FUSE_EXPAND) on C2 / C5 / C3, alternating runs on one box,
# plus the contract tests that cover it.
set -x
mkdir -p gpurun_out/fuse
python -m pytest tests/test_gpu_contracts.py -q -x -k "variants or merged" 2>&1 | tail -3 > gpurun_out/fuse/pytest.log
for r in 1 2; do
  for f in 1 0; do
    HSDLA_FUSE_EXPAND=$f python bench.py --steps 20 --no-extras --no-cpu-baseline > gpurun_out/fuse/C2_f${f}_r$r.json 2> gpurun_out/fuse/C2_f${f}_r$r.err
    HSDLA_FUSE_EXPAND=$f python bench.py --config C5 --steps 20 --no-extras --no-cpu-baseline > gpurun_out/fuse/C5_f${f}_r$r.json 2> gpurun_out/fuse/C5_f${f}_r$r.err
  done
done
for f in 1 0; do
  HSDLA_FUSE_EXPAND=$f python bench.py --config C3 --steps 5 --no-extras --no-cpu-baseline > gpurun_out/fuse/C3_f${f}.json 2> gpurun_out/fuse/C3_f${f}.err
done
CMD="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/fuse/launches_C2.csv $CMD > /dev/null 2>&1
ls gpurun_out/fuse
