# try_wait vs non-suspending test_wait polls in the variance rings (skeleton and complete kernels)
mkdir -p gpurun_out/sp; : > gpurun_out/sp/sum.log
L=$PWD/paper_2411_03289_b200/lib
for c in config2 config5; do for lib in diag diagspin; do for pair in 0 1; do for d in 0 261 257; do
  GPMPPI_LIB=$L/libgpmppi_b200_$lib.so GPMPPI_VAR2CTA=$pair GPMPPI_TC_DEBUG=$d timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 2 > gpurun_out/sp/b.json 2>&1
  echo "[$c $lib pair=$pair dbg=$d] $(python -c "import json; d=json.loads(open('gpurun_out/sp/b.json').read().strip().splitlines()[-1]); print(round(d['phase_ms']['variance'],4))" 2>&1 | tail -1)" >> gpurun_out/sp/sum.log
done; done; done; done
