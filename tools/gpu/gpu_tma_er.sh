# The TMA kernel's K loop in the early-reload order: parity (it carries the per-type W application by
# default, and every contraction with HSDLA_CONTRACT=tma), then C2 / C3 bench lines default vs all-TMA.
mkdir -p gpurun_out/tmaer
python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py tests/test_gpu_joint.py -m gpu -q -x 2>&1 | tail -1
HSDLA_CONTRACT=tma python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden_big.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
  for c in C2 C3; do
    python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/tmaer/${c}_default_r$r.json 2>/dev/null
    HSDLA_CONTRACT=tma python bench.py --config $c --steps 10 --no-extras --no-cpu-baseline > gpurun_out/tmaer/${c}_alltma_r$r.json 2>/dev/null
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/tmaer/*_r*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], d["ms_per_step"], d["fp64_peak_frac"], d["roofline"]["contract_ms_per_step"], d["roofline"]["kernel_ms"].get("apply_W"))
    except Exception as e: print(f, "ERR", e)
P
