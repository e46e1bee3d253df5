# Round-2 evidence pass after the K-loop reordering (early fragment reload, cp.async block under the first loads):
# same recipe as gpu_evidence_r02b.sh / r02c.sh.
set -x
mkdir -p gpurun_out/ev8
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev8/pytest_gpu_1.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev8/smoke.log 2>&1
python bench.py > gpurun_out/ev8/bench_C2.json 2> gpurun_out/ev8/bench_C2.err
for c in C3 C4 C5 C2NS C2IND C1; do
  python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/ev8/bench_$c.json 2> gpurun_out/ev8/bench_$c.err
done
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ev8/bench_ref_C2.json 2> gpurun_out/ev8/bench_ref_C2.err
python bench.py --mode panels --config C4 --steps 3 > gpurun_out/ev8/bench_panels_C4.json 2> gpurun_out/ev8/bench_panels_C4.err
CMD="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
$CMD > gpurun_out/ev8/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ev8/launches_C2.csv $CMD > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:contract -c 8 --clock-control none --csv --log-file gpurun_out/ev8/traffic_C2.csv python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"contract_kernel" -s 4 -c 1 -o gpurun_out/ev8/ncu_SH_C2 $CMD > /dev/null 2>&1
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev8/pytest_gpu_2.log
ls gpurun_out/ev8
