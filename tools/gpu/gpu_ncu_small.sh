# ncu --set full of the small per-k-point kernels on C2 (template generator, expansion, W
# application), for the generator-path analysis.
mkdir -p gpurun_out/ncusmall
CMD="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ab_kernel|expand_kernel|contract_tma" -s 9 -c 3 -o gpurun_out/ncusmall/small $CMD > gpurun_out/ncusmall/ncu.log 2>&1
ls -la gpurun_out/ncusmall
