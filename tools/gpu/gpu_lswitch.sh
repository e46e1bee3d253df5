# Copy-bound synchronous calls: L pieces for the first tile columns, then truncated panels
# (HSDLA_LSWITCH tile columns; 0 = panels only); streamed-copy tests.
mkdir -p gpurun_out/ls
python -m pytest tests/test_gpu_contracts.py -m gpu -q -k "streamed_copy" 2>&1 | tail -2 > gpurun_out/ls/pytest.log
for r in 1 2; do
  for v in 0 def 8 24; do
    E="HSDLA_LSWITCH=$v"; [ $v = def ] && E="HSDLA_X=1"
    env $E python tools/copy_timeline.py C2 > gpurun_out/ls/C2_${v}_r$r.txt 2>&1
  done
done
