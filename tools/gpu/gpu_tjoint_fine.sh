mkdir -p gpurun_out/tja
for m in 81 40; do tools/exp/tjoint_bench_192 $m | tail -1; done > gpurun_out/tja/fine.log 2>&1
