set -x
mkdir -p gpurun_out/single
python tools/pcie_probe.py > gpurun_out/single/pcie.txt 2>&1
for g in 1 2 4 8 47; do
HSDLA_COPY_PANELS=$g python tools/copy_timeline.py C2 > gpurun_out/single/timeline_$g.txt 2>&1
done
