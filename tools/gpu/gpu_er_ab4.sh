# A/B of K-loop order variants on top of the early-reload default: er3 = cp.async block issued after the
# chunk's first fragment loads, er4 = sums formed right before their first use, er5 = mirror order (row
# block outer, column fragments carried).  Parity subset per variant, then alternating bench runs.
mkdir -p gpurun_out/er4
for v in er3 er4 er5; do
  HSDLA_LIB=$PWD/tools/exp/libhsdla_$v.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py -m gpu -q -x 2>&1 | tail -1 > gpurun_out/er4/pytest_$v.log
  cat gpurun_out/er4/pytest_$v.log
done
for r in 1 2; do
  for c in C2 C3; do
    for v in head er3 er4 er5; do
      if [ $v = head ]; then L=""; else L=$PWD/tools/exp/libhsdla_$v.so; fi
      HSDLA_LIB=$L python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/er4/${c}_${v}_r$r.json 2>/dev/null
    done
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/er4/*_r*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], d["ms_per_step"], d["fp64_peak_frac"], d["roofline"]["contract_ms_per_step"])
    except Exception as e: print(f, "ERR", e)
P
