# A/B of the variance phase: default library vs lib/libgpmppi_b200_$VAR.so, single-CTA and CTA-pair kernels
mkdir -p gpurun_out/p9; SUM=gpurun_out/p9/sum_${CONFIG:-config2}.log; : > $SUM
for rep in 1 2; do for lib in "" "$PWD/paper_2411_03289_b200/lib/libgpmppi_b200_${VAR}.so"; do for pair in ${PAIRS:-0 1}; do for d in ${DBGS:-0}; do
  GPMPPI_LIB=${lib:-$DEFLIB} GPMPPI_VAR2CTA=$pair GPMPPI_TC_DEBUG=$d timeout 300 python bench.py --config ${CONFIG:-config2} --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 2 > gpurun_out/p9/b.json 2>&1
  echo "[lib=${lib:+$VAR} pair=$pair dbg=$d] $(python -c "import json; d=json.loads(open('gpurun_out/p9/b.json').read().strip().splitlines()[-1]); print(round(d['phase_ms']['variance'],4))" 2>&1 | tail -1)" >> $SUM
done; done; done; done
