# ncu launch list (per-launch device time) of a short C2 bench run.
CMD="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_C2.csv $CMD > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
