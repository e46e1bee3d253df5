# A/B of the contraction's sum-plane ring variants on C2 (bench lines into gpurun_out/).
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 8x4 8x3 16x2; do
  HSDLA_PL_VARIANT=$v python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/plv_$v.json 2>&1
done
HSDLA_PLANES=0 python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/plv_off.json 2>&1
for f in plv_8x4 plv_8x3 plv_16x2 plv_off; do
  python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['ab_gen']['ms'])"
done
