mkdir -p gpurun_out/c3; : > gpurun_out/c3/sum.log
for rep in 1 2; do for v in "" 0 1; do
  env ${v:+GPMPPI_VAR2CTA=$v} timeout 300 python bench.py --config ${CONFIG:-config3} --steps 5 --warmup 3 --no-cpu-baseline --e2e-ticks 2 > gpurun_out/c3/b.json 2>&1
  echo "[VAR2CTA=${v:-auto}] $(python -c "import json; d=json.loads(open('gpurun_out/c3/b.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['phase_ms']['variance'],4), d['roofline']['kernels'].keys())" 2>&1 | tail -1)" >> gpurun_out/c3/sum.log
done; done
