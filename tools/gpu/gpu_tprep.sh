# ncu launch list of the T preparation kernels on first builds (tools/tprep_probe.py).
python tools/tprep_probe.py > gpurun_out/tprep_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tjoint|tprep" --csv \
    --log-file gpurun_out/tprep_launches.csv python tools/tprep_probe.py > gpurun_out/tprep_ncu.log 2>&1
cat gpurun_out/tprep_plain.log
grep -E "tjoint|tprep" gpurun_out/tprep_launches.csv | awk -F'","' '{print $5, $(NF)}' | cut -c1-150
