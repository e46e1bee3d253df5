# Final check after the last code change (per-group copy counters): GPU suite, smoke, bench
# lines of the configs whose single-call numbers moved.
mkdir -p gpurun_out/fin
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/fin/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1
python bench.py > gpurun_out/fin/bench_C2.json 2> gpurun_out/fin/bench_C2.err
for c in C3 C5 C2IND C2NS; do
  python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/fin/bench_$c.json 2> gpurun_out/fin/bench_$c.err
done
