# A/B: DMMA asm volatile (default build) vs register-only asm (tools/exp/libhsdla_nv.so).
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/nv_def.json 2>&1
HSDLA_LIB=$PWD/tools/exp/libhsdla_nv.so python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/nv_nv.json 2>&1
HSDLA_LIB=$PWD/tools/exp/libhsdla_nv.so python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for f in nv_def nv_nv; do
  python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['ab_gen']['ms'])"
done
