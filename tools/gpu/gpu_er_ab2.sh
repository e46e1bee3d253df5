# A/B of early-reload variants ER=1 / ER=2 (tools/exp/libhsdla_er.so, libhsdla_er2.so) against the default library.
mkdir -p gpurun_out/er2
for r in 1 2; do
  for c in C2 C3; do
    for v in head er er2; do
      if [ $v = head ]; then L=""; else L=$PWD/tools/exp/libhsdla_$v.so; fi
      HSDLA_LIB=$L python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/er2/${c}_${v}_r$r.json 2>/dev/null
    done
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/er2/*_r*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], d["ms_per_step"], d["fp64_peak_frac"], d["roofline"]["contract_ms_per_step"])
    except Exception as e: print(f, "ERR", e)
P
