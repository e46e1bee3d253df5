# Streamed copies of synchronous calls, L vs panel shapes (HSDLA_LCOPY), by config; GPU suite.
mkdir -p gpurun_out/lc3
python tools/copy_timeline.py C2 > gpurun_out/lc3/timeline_C2.txt 2>&1
HSDLA_LCOPY=1 python tools/copy_timeline.py C2 > gpurun_out/lc3/timeline_C2_L.txt 2>&1
for c in C2 C3 C5 C4; do
  python bench.py --config $c --steps 3 --no-extras --no-cpu-baseline > gpurun_out/lc3/$c.json 2> gpurun_out/lc3/$c.err
done
HSDLA_LCOPY=0 python bench.py --config C5 --steps 3 --no-extras --no-cpu-baseline > gpurun_out/lc3/C5_panels.json 2> gpurun_out/lc3/C5_panels.err
python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/lc3/pytest.log
