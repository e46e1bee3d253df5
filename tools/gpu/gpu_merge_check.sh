set -x
mkdir -p gpurun_out/mck
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/mck/pytest.log
python bench.py --steps 30 --no-extras --no-cpu-baseline > gpurun_out/mck/C2.json 2> gpurun_out/mck/C2.err
python bench.py --config C5 --steps 30 --no-extras --no-cpu-baseline > gpurun_out/mck/C5.json 2> gpurun_out/mck/C5.err
