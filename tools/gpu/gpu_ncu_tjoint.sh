# ncu --set full of the first tjoint_kernel (C2) launched by tools/tprep_probe.py
python tools/tprep_probe.py C2 > gpurun_out/tprep_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tjoint" -c 1 -o gpurun_out/r02_tjoint python tools/tprep_probe.py C2 > gpurun_out/ncu_tj.log 2>&1
tail -2 gpurun_out/ncu_tj.log
