# A/B: the default three-product kernel compiled without the runtime spread code (er10) against the default.
mkdir -p gpurun_out/er7
HSDLA_LIB=$PWD/tools/exp/libhsdla_er10.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
  for c in C2 C3 C5; do
    for v in head er10; do
      L=""
      if [ $v = er10 ]; then L=$PWD/tools/exp/libhsdla_$v.so; fi
      HSDLA_LIB=$L python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/er7/${c}_${v}_r$r.json 2>/dev/null
    done
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/er7/*_r*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], d["ms_per_step"], d["fp64_peak_frac"], d["roofline"]["contract_ms_per_step"])
    except Exception as e: print(f, "ERR", e)
P
