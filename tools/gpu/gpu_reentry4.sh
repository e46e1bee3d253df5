# Re-entry check of HEAD in a re-created container: GPU suite, smoke, the driver's two bench arms.
mkdir -p gpurun_out/re4
python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/re4/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re4/smoke.log 2>&1
python bench.py > gpurun_out/re4/bench_C2.json 2> gpurun_out/re4/bench_C2.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/re4/bench_ref_C2.json 2> gpurun_out/re4/bench_ref_C2.err
python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/re4/bench_g2.json 2> gpurun_out/re4/bench_g2.err
cat gpurun_out/re4/pytest_gpu.log gpurun_out/re4/smoke.log
