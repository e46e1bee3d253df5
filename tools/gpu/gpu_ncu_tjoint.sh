# ncu --set full of the first tjoint_kernel (C2) launched by tools/tprep_probe.py
mkdir -p gpurun_out/tjn
python tools/tprep_probe.py C2 > gpurun_out/tjn/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tjoint" -c 1 -o gpurun_out/tjn/tjoint python tools/tprep_probe.py C2 > gpurun_out/tjn/ncu.log 2>&1
tail -2 gpurun_out/tjn/ncu.log
