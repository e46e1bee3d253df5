# A/B on top of the new default (early reload + cp.async block under the first fragment loads):
# er5 = mirror order (row block outer) with the same cp.async placement, er7 = the previous default
# (cp.async block right after the barrier), plus HSDLA_CP_SPREAD=1 on the default.
mkdir -p gpurun_out/er5
HSDLA_LIB=$PWD/tools/exp/libhsdla_er5.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
  for c in C2 C3; do
    for v in head er5 er7 spread; do
      L=""; SP=0
      if [ $v = er5 ] || [ $v = er7 ]; then L=$PWD/tools/exp/libhsdla_$v.so; fi
      if [ $v = spread ]; then SP=1; fi
      HSDLA_CP_SPREAD=$SP HSDLA_LIB=$L python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/er5/${c}_${v}_r$r.json 2>/dev/null
    done
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/er5/*_r*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], d["ms_per_step"], d["fp64_peak_frac"], d["roofline"]["contract_ms_per_step"])
    except Exception as e: print(f, "ERR", e)
P
