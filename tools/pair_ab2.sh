mkdir -p gpurun_out/p8; : > gpurun_out/p8/sum.log
nvidia-smi --query-gpu=name,serial --format=csv >> gpurun_out/p8/sum.log
for rep in 1 2; do for lib in "" "$PWD/paper_2411_03289_b200/lib/libgpmppi_b200_notrace.so"; do for pair in 0 1; do
  GPMPPI_TC_PRINT=1 GPMPPI_LIB=$lib GPMPPI_VAR2CTA=$pair timeout 300 python bench.py --config config2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 2 > gpurun_out/p8/b.json 2>&1
  echo "[lib=${lib:+notrace} pair=$pair] $(grep -m1 pairs gpurun_out/p8/b.json) $(python -c "import json; d=json.loads(open('gpurun_out/p8/b.json').read().strip().splitlines()[-1]); print(round(d['phase_ms']['variance'],4))" 2>&1 | tail -1)" >> gpurun_out/p8/sum.log
done; done; done
