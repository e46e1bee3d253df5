# Re-entry check of HEAD on a fresh box: GPU suite, smoke, C2 bench line.
set -x
mkdir -p gpurun_out/r02c
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r02c/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c/smoke.log 2>&1
python bench.py > gpurun_out/r02c/bench_C2.json 2> gpurun_out/r02c/bench_C2.err
python bench.py --config C3 --steps 5 --no-extras --no-cpu-baseline > gpurun_out/r02c/bench_C3.json 2> gpurun_out/r02c/bench_C3.err
ls gpurun_out/r02c
