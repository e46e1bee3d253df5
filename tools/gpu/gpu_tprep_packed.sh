# Packed shared-memory T factorisations vs the blocked global-memory ones: GPU suite parts that
# exercise the T preparation, then ncu launch lists of first builds (tools/tprep_probe.py C2).
mkdir -p gpurun_out/tp
python -m pytest tests/test_gpu_joint.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_contracts.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/tp/pytest.log
for v in 1 0; do
  HSDLA_TPREP_PACKED=$v python tools/tprep_probe.py C2 > gpurun_out/tp/plain_$v.log 2>&1 && \
  HSDLA_TPREP_PACKED=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tjoint|tprep" --csv \
      --log-file gpurun_out/tp/launches_$v.csv python tools/tprep_probe.py C2 > gpurun_out/tp/ncu_$v.log 2>&1
done
