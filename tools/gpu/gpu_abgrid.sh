# Per-atom A/B generator with atoms fastest vs HEAD (C2NS per-atom path; the drop-in compute_AB),
# alternating; A/B parity tests.
mkdir -p gpurun_out/abg
python -m pytest tests/test_gpu_parity.py tests/test_gpu_special.py tests/test_gpu_edges.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/abg/pytest.log
for r in 1 2; do
  for v in head new; do
    L=""; [ $v = head ] && L="HSDLA_LIB=ab/libhsdla_head.so"
    env $L python bench.py --config C2NS --steps 10 --no-extras --no-cpu-baseline > gpurun_out/abg/C2NS_${v}_r$r.json 2>/dev/null
    env $L HSDLA_TEMPLATES=0 python bench.py --config C3 --steps 3 --no-extras --no-cpu-baseline > gpurun_out/abg/C3pa_${v}_r$r.json 2>/dev/null
  done
done
