# Expansion kernel A/B: HEAD library vs working tree, alternating; template-path parity.
mkdir -p gpurun_out/ex5
python -m pytest tests/test_gpu_joint.py tests/test_gpu_parity.py tests/test_gpu_golden_big.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/ex5/pytest.log
for c in C2 C3 C5 C4; do
  for r in 1 2; do
    HSDLA_LIB=ab/libhsdla_head.so python bench.py --config $c --steps 3 --no-extras --no-cpu-baseline > gpurun_out/ex5/${c}_head_r$r.json 2>/dev/null
    python bench.py --config $c --steps 3 --no-extras --no-cpu-baseline > gpurun_out/ex5/${c}_new_r$r.json 2>/dev/null
  done
done
