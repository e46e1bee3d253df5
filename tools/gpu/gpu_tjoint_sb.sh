# blocked Cholesky panel step size (HSDLA_CHOL_SB) and rsqrt pivots (HSDLA_CHOL_RSQRT) in the joint T factor phase harness
mkdir -p gpurun_out/tja
for m in 81 40 121; do for v in sb4_r0 sb4_r1 sb8_r0 sb8_r1; do echo "== $v m=$m"; tools/exp/tjoint_$v $m | tail -2; done; done > gpurun_out/tja/sb.log 2>&1
