#!/bin/bash
# FP64 ceiling probe under gpurun: DMMA/DFMA microbench + cuBLAS, clocks sampled alongside.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/fp64_probe > gpurun_out/fp64_probe.log 2>&1
python tools/cublas_fp64_ceiling.py > gpurun_out/cublas_fp64.log 2>&1
kill $SMI
nvidia-smi > gpurun_out/nvidia_smi.txt
cat gpurun_out/fp64_probe.log gpurun_out/cublas_fp64.log
