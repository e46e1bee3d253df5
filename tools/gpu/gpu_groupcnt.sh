# One tile counter per copy group (one stream wait per copy) vs HEAD's per-column counters:
# streamed-copy tests, single-call timelines C2 / C5 alternating with the HEAD library.
mkdir -p gpurun_out/gc
python -m pytest tests/test_gpu_contracts.py -m gpu -q -k "streamed_copy or merged" 2>&1 | tail -2 > gpurun_out/gc/pytest.log
for r in 1 2; do
  for v in head new; do
    L=""; [ $v = head ] && L="HSDLA_LIB=ab/libhsdla_head.so"
    env $L python tools/copy_timeline.py C2 > gpurun_out/gc/C2_${v}_r$r.txt 2>&1
    env $L python tools/copy_timeline.py C5 2>&1 | grep wall | tail -2 > gpurun_out/gc/C5_${v}_r$r.txt
  done
done
