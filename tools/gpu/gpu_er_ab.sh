# A/B of the early-reload contraction variant (tools/exp/libhsdla_er.so, `make -C paper_1602_06589_b200/csrc er`)
# against the default library: parity subset with the variant, then alternating bench runs.
mkdir -p gpurun_out/er
HSDLA_LIB=$PWD/tools/exp/libhsdla_er.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py tests/test_gpu_golden_big.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/er/pytest_er.log
cat gpurun_out/er/pytest_er.log
for r in 1 2; do
  for c in C2 C3 C5; do
    python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/er/${c}_head_r$r.json 2>/dev/null
    HSDLA_LIB=$PWD/tools/exp/libhsdla_er.so python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/er/${c}_er_r$r.json 2>/dev/null
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/er/*_r*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], d["ms_per_step"], d["fp64_peak_frac"], d["roofline"]["contract_ms_per_step"])
    except Exception as e: print(f, "ERR", e)
P
