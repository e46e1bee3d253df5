# T preparation after the register row sums (joint assembly) and the single-thread diagonal block factor:
# GPU tests touching the Cholesky / joint paths, and the first-build launch list (tprep / tjoint) of C2 and C4.
mkdir -p gpurun_out/tpc
python -m pytest tests/test_gpu_joint.py tests/test_gpu_contracts.py tests/test_gpu_parity.py tests/test_gpu_special.py -q -x 2>&1 | tail -3 > gpurun_out/tpc/pytest.log
python tools/tprep_probe.py C2 C4 > gpurun_out/tpc/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tprep|tjoint" --csv --log-file gpurun_out/tpc/launches.csv python tools/tprep_probe.py C2 C4 > /dev/null 2>&1
