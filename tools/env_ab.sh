# A/B of the variance phase over environment settings: ENVS="A=1;A=2" (";"-separated), CONFIGS
mkdir -p gpurun_out/ea; SUM=gpurun_out/ea/sum.log; : > $SUM
IFS=';' read -ra SETS <<< "${ENVS:-GPMPPI_F16_CPS=1;GPMPPI_F16_CPS=2}"
for c in ${CONFIGS:-config2 config5}; do for rep in 1 2; do for e in "${SETS[@]}"; do
  env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 2 > gpurun_out/ea/b.json 2>&1
  echo "[$c $e] $(python -c "import json; d=json.loads(open('gpurun_out/ea/b.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['phase_ms']['variance'],4))" 2>&1 | tail -1)" >> $SUM
done; done; done
