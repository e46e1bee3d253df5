# Streamed copy shapes: panels (0), L (1), L with batched mirror rows (2); alternating repeats.
mkdir -p gpurun_out/lb2
python -m pytest tests/test_gpu_contracts.py -m gpu -q -k streamed_copy 2>&1 | tail -2 > gpurun_out/lb2/pytest_default.log
HSDLA_LCOPY=2 python -m pytest tests/test_gpu_contracts.py -m gpu -q -k "streamed_copy and not LCOPY" 2>&1 | tail -2 > gpurun_out/lb2/pytest_l2.log
for r in 1 2; do
  for v in 0 1 2; do
    HSDLA_LCOPY=$v python tools/copy_timeline.py C2 2>&1 | grep wall | tail -2 > gpurun_out/lb2/C2_l${v}_r$r.txt
    HSDLA_LCOPY=$v python tools/copy_timeline.py C5 2>&1 | grep wall | tail -2 > gpurun_out/lb2/C5_l${v}_r$r.txt
  done
done
HSDLA_LCOPY=2 python tools/copy_timeline.py C2 > gpurun_out/lb2/timeline_C2_l2.txt 2>&1
for v in 1 2; do
  HSDLA_LCOPY=$v python tools/copy_timeline.py C3 2>&1 | grep wall | tail -2 > gpurun_out/lb2/C3_l${v}.txt
done
