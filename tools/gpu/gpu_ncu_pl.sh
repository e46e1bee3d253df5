set -e
CMD="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"contract_kernel" -s 6 -c 1 -o gpurun_out/r02_pl_S $CMD > gpurun_out/ncu1.log 2>&1
HSDLA_PLANES=0 ncu --set full --clock-control none --import-source on -k regex:"contract_kernel" -s 6 -c 1 -o gpurun_out/r02_g3_S $CMD > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu1.log gpurun_out/ncu2.log
