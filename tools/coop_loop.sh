# repeat tools/coopdbg.py under several settings, count failures and record the first error line
mkdir -p gpurun_out/r2n; : > gpurun_out/r2n/sum.log
for cfg in "" "DBG_OBS=10" "GPMPPI_NO_GRAPH=1"; do
  fails=0; first=""
  for i in 1 2 3 4 5 6 7 8; do
    env DBG_OBS=0 $cfg timeout 60 python tools/coopdbg.py combined philox > gpurun_out/r2n/g.log 2>&1
    if [ $? -ne 0 ]; then fails=$((fails+1)); [ -z "$first" ] && first="$(grep -m1 CudaError gpurun_out/r2n/g.log | cut -c1-160)"; fi
  done
  echo "$cfg -> fails $fails/8 $first" >> gpurun_out/r2n/sum.log
done
