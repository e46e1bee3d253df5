# A/B of contraction warp layouts on C2 (bench lines into gpurun_out/).
run() { name=$1; shift; env "$@" python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/wv_$name.json 2>&1;
  python -c "import json; d=json.loads(open('gpurun_out/wv_$name.json').read().strip().splitlines()[-1]); print('$name', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])" || tail -3 gpurun_out/wv_$name.json; }
run def HSDLA_X=0
run jb2m1 HSDLA_WARP_COLS=16
run jb2m2 HSDLA_WARP_COLS=16 HSDLA_G3_MINB=2
run tma4 HSDLA_CONTRACT=tma
run tma8 HSDLA_CONTRACT=tma HSDLA_TMA_W8=1
HSDLA_WARP_COLS=16 HSDLA_G3_MINB=2 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
HSDLA_CONTRACT=tma HSDLA_TMA_W8=1 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
