# joint T factor phase split (tools/exp_tjoint_bench.cu): HEAD assembly (shared-memory double atomics per element) vs
# register row sums, one CTA (cluster from 2m >= 192) vs cluster forced (HSDLA_CLUSTER_MIN_N=0); m = 81 (C2), 121 (C4), 40.
mkdir -p gpurun_out/tja
for m in 81 121 40; do
  for b in head 192 0; do
    echo "== $b m=$m" >> gpurun_out/tja/out.log
    tools/exp/tjoint_bench_$b $m >> gpurun_out/tja/out.log 2>&1
  done
done
