# A/B on top of the default (early reload + cp.async block under the first fragment loads): er8 = the cp.async
# block in two halves (after the first loads / before K group 1), er9 = the whole block before K group 1,
# plus HSDLA_CP_SPREAD=1.
mkdir -p gpurun_out/er6
HSDLA_LIB=$PWD/tools/exp/libhsdla_er8.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py -m gpu -q -x 2>&1 | tail -1
HSDLA_LIB=$PWD/tools/exp/libhsdla_er9.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
  for c in C2 C3; do
    for v in head er8 er9; do
      L=""; SP=0
      if [ $v = er8 ] || [ $v = er9 ]; then L=$PWD/tools/exp/libhsdla_$v.so; fi
      if [ $v = spread ]; then SP=1; fi
      HSDLA_CP_SPREAD=$SP HSDLA_LIB=$L python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/er6/${c}_${v}_r$r.json 2>/dev/null
    done
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/er6/*_r*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], d["ms_per_step"], d["fp64_peak_frac"], d["roofline"]["contract_ms_per_step"])
    except Exception as e: print(f, "ERR", e)
P
