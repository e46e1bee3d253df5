set -x
mkdir -p gpurun_out/mck2
nvidia-smi -q | grep -i -A3 "PCI\b\|Link Width\|Max Link Gen\|Current Link Gen" | head -30 > gpurun_out/mck2/pci.txt
for rep in 1 2; do
for m in 1 0; do
HSDLA_MERGE_SH=$m python bench.py --steps 30 --no-extras --no-cpu-baseline > gpurun_out/mck2/C2_m${m}_$rep.json 2> gpurun_out/mck2/C2_m${m}_$rep.err
done
done
