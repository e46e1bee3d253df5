# A/B of the chunk-carry variant (ER=2, tools/exp/libhsdla_er.so) against the default library (early reload inside a chunk).
mkdir -p gpurun_out/er3
HSDLA_LIB=$PWD/tools/exp/libhsdla_er.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py tests/test_gpu_golden_big.py tests/test_gpu_edges.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/er3/pytest_er.log
cat gpurun_out/er3/pytest_er.log
for r in 1 2; do
  for c in C2 C3; do
    for v in head er; do
      if [ $v = head ]; then L=""; else L=$PWD/tools/exp/libhsdla_$v.so; fi
      HSDLA_LIB=$L python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/er3/${c}_${v}_r$r.json 2>/dev/null
    done
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/er3/*_r*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], d["ms_per_step"], d["fp64_peak_frac"], d["roofline"]["contract_ms_per_step"])
    except Exception as e: print(f, "ERR", e)
P
