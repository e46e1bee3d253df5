# Sanity pass after a container rebuild: full GPU suite, default bench line.
mkdir -p gpurun_out/san
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/san/pytest_gpu.log
python bench.py > gpurun_out/san/bench_C2.json 2> gpurun_out/san/bench_C2.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/smoke.log 2>&1
