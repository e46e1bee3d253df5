# Expansion kernel A/B: HEAD library (2-D grid, one atom per CTA) vs working tree (per type).
mkdir -p gpurun_out/ex3
python tools/hbm_write_probe.py > gpurun_out/ex3/write_probe.txt 2>&1
for c in C2 C3 C5; do
  HSDLA_LIB=ab/libhsdla_head.so python bench.py --config $c --steps 5 --no-extras --no-cpu-baseline > gpurun_out/ex3/${c}_head.json 2>/dev/null
  python bench.py --config $c --steps 5 --no-extras --no-cpu-baseline > gpurun_out/ex3/${c}_new.json 2>/dev/null
done
