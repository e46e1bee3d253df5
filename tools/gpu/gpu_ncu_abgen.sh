# ncu --set full with source of the per-type template generator (ab_kernel<8>, zero_phase) on C2.
mkdir -p gpurun_out/ncuab
CMD="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ab_kernel" -s 3 -c 1 -o gpurun_out/ncuab/ab $CMD > gpurun_out/ncuab/ncu.log 2>&1
