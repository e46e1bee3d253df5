# ncu --set full with SASS source of the C2 S contraction (default kernel), for stall analysis.
mkdir -p gpurun_out/ncuS
CMD="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
$CMD > gpurun_out/ncuS/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"contract_kernel" -s 6 -c 1 -o gpurun_out/ncuS/S_C2 $CMD > gpurun_out/ncuS/ncu.log 2>&1
ls -la gpurun_out/ncuS
