# Warp-per-K template generator (HSDLA_AB_TPL=1) vs the per-thread kernel: bitwise H / S on C2
# and C5 builds (dumps in /tmp, only the verdicts come back); template-path tests; bench lines.
mkdir -p gpurun_out/at /tmp/at
for c in C2 C5 C1; do
  HSDLA_AB_TPL=0 python tools/tpl_bitwise.py $c /tmp/at/${c}_0.npz
  HSDLA_AB_TPL=1 python tools/tpl_bitwise.py $c /tmp/at/${c}_1.npz
  python -c "
import numpy as np
a=np.load('/tmp/at/${c}_0.npz'); b=np.load('/tmp/at/${c}_1.npz')
print('$c', 'types', int(a['types']), int(b['types']), 'H bitwise', np.array_equal(a['h'], b['h']), 'S bitwise', np.array_equal(a['s'], b['s']))
" >> gpurun_out/at/bitwise.txt 2>&1
done
rm -rf /tmp/at
python -m pytest tests/test_gpu_joint.py tests/test_gpu_parity.py tests/test_gpu_golden_big.py tests/test_gpu_edges.py tests/test_gpu_contracts.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/at/pytest.log
for r in 1 2; do
  for v in 0 1; do
    HSDLA_AB_TPL=$v python bench.py --steps 20 --no-extras --no-cpu-baseline > gpurun_out/at/C2_${v}_r$r.json 2>/dev/null
    HSDLA_AB_TPL=$v python bench.py --config C5 --steps 5 --no-extras --no-cpu-baseline > gpurun_out/at/C5_${v}_r$r.json 2>/dev/null
  done
done
